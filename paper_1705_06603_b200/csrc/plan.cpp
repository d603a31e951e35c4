// plan.cpp -- facet planner (see plan.hpp for the readings it implements).
#include "plan.hpp"

#include <algorithm>
#include <limits>
#include <sstream>

namespace deblur {

std::string axis_plan(int64_t M, int F, int O, int P, std::vector<AxisFacet> &out) {
    out.clear();
    if (F < 1) return "facet grid must be >= 1 per axis";
    if (O < 0 || (O % 2) != 0) return "overlap must be even and >= 0";
    if (M < F) return "observed extent smaller than the facet count";
    for (int k = 0; k < F; ++k) {
        int64_t b0 = (int64_t)k * M / F, b1 = (int64_t)(k + 1) * M / F;
        int64_t lo = (k == 0) ? 0 : std::max<int64_t>(0, b0 - O / 2);
        int64_t hi = (k == F - 1) ? M : std::min<int64_t>(M, b1 + O / 2);
        out.push_back({lo, hi, lo, hi + P - 1});
    }
    for (int k = 1; k + 1 < F; ++k)
        if (out[k - 1].e_hi > out[k + 1].e_lo) {
            std::ostringstream s;
            s << "facet " << k << " core too small: estimate bands of facets " << k - 1 << " and " << k + 1
              << " overlap (need facet core >= overlap + P - 1)";
            return s.str();
        }
    return "";
}

static int64_t cut_cost(int gy, int gx, int64_t ny, int64_t nx) {
    return (int64_t)(gy - 1) * nx + (int64_t)(gx - 1) * ny;
}

std::string make_plan(int64_t ny, int64_t nx, int P, int Fy, int Fx, int O, int world, Plan &pl) {
    pl = Plan();
    if (P < 1 || (P % 2) == 0) return "psf_size must be odd and >= 1";
    if (P > ny || P > nx) return "psf_size larger than the image";
    pl.ny = ny; pl.nx = nx; pl.P = P; pl.Fy = Fy; pl.Fx = Fx; pl.O = O;
    pl.my = ny - P + 1; pl.mx = nx - P + 1;
    std::string e = axis_plan(pl.my, Fy, O, P, pl.ay);
    if (!e.empty()) return "rows: " + e;
    e = axis_plan(pl.mx, Fx, O, P, pl.ax);
    if (!e.empty()) return "cols: " + e;
    // GPU grid: g_y | F_y, g_x | F_x, g_y*g_x == world, minimum cut length
    if (world < 1) return "world must be >= 1";
    int best_y = -1;
    int64_t best = std::numeric_limits<int64_t>::max();
    for (int g = 1; g <= world; ++g) {
        if (world % g) continue;
        int h = world / g;
        if (Fy % g || Fx % h) continue;
        int64_t c = cut_cost(g, h, ny, nx);
        if (c < best) { best = c; best_y = g; }
    }
    if (best_y < 0) {
        std::ostringstream s;
        s << "world " << world << " does not factor into a GPU grid dividing the " << Fy << "x" << Fx << " facet grid";
        return s.str();
    }
    pl.gy = best_y; pl.gx = world / best_y;
    const int fpy = Fy / pl.gy, fpx = Fx / pl.gx;
    for (int a = 0; a < Fy; ++a)
        for (int b = 0; b < Fx; ++b) {
            FacetPlan f;
            f.id = a * Fx + b; f.fy = a; f.fx = b;
            f.owner = (a / fpy) * pl.gx + (b / fpx);
            f.oy0 = pl.ay[a].o_lo; f.oy1 = pl.ay[a].o_hi; f.ox0 = pl.ax[b].o_lo; f.ox1 = pl.ax[b].o_hi;
            f.ey0 = pl.ay[a].e_lo; f.ey1 = pl.ay[a].e_hi; f.ex0 = pl.ax[b].e_lo; f.ex1 = pl.ax[b].e_hi;
            f.py_e = (a > 0) ? pl.ay[a - 1].e_hi : f.ey0;
            f.ny_s = (a + 1 < Fy) ? pl.ay[a + 1].e_lo : f.ey1;
            f.px_e = (b > 0) ? pl.ax[b - 1].e_hi : f.ex0;
            f.nx_s = (b + 1 < Fx) ? pl.ax[b + 1].e_lo : f.ex1;
            pl.facets.push_back(f);
            if (f.oy1 - f.oy0 < 2 * P || f.ox1 - f.ox0 < 2 * P) {
                std::ostringstream s;
                s << "facet " << f.id << " observed block " << (f.oy1 - f.oy0) << "x" << (f.ox1 - f.ox0)
                  << " is smaller than twice the PSF (PAPER.md:259)";
                pl.warnings.push_back(s.str());
            }
        }
    return "";
}

Rect overlap(const FacetPlan &a, const FacetPlan &b) {
    Rect r{std::max(a.ey0, b.ey0), std::min(a.ey1, b.ey1), std::max(a.ex0, b.ex0), std::min(a.ex1, b.ex1)};
    if (a.id == b.id || r.empty()) return Rect{0, 0, 0, 0};
    return r;
}

std::vector<Message> messages_from(const Plan &pl, int rank) {
    std::vector<Message> out;
    for (const auto &d : pl.facets)
        for (const auto &s : pl.facets) {
            if (s.owner != rank || d.owner == rank) continue;
            Rect r = overlap(s, d);
            if (r.empty()) continue;
            out.push_back({d.owner, s.id, d.id, r});
        }
    return out;
}

std::vector<Message> messages_to(const Plan &pl, int rank) {
    std::vector<Message> out;
    for (const auto &d : pl.facets)
        for (const auto &s : pl.facets) {
            if (d.owner != rank || s.owner == rank) continue;
            Rect r = overlap(s, d);
            if (r.empty()) continue;
            out.push_back({s.owner, s.id, d.id, r});
        }
    return out;
}

}  // namespace deblur
