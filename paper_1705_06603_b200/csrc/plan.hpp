// plan.hpp -- host-side facet planner for libdeblur (no CUDA dependencies).
//
// Readings (SURVEY.md §8c / DESIGN.md §2):
//   A12  overlap O between OBSERVED blocks; b_k = floor(k*M/F); O_f =
//        [b_f - O/2, b_{f+1} + O/2) clipped; P_f = O_f dilated by (P-1)/2 on
//        each side (PAPER.md:118 index sets, :239 extra boundary pixels)
//   A13  consensus weights: ramp (t - s + 0.5)/(e - s) on each shared band
//        (PAPER.md:206 alpha = gamma*omega, Fig. 1 ramp :239)
//   A28  8-neighbour halo exchange (a pixel may lie in 4 blocks)
//   §8e  facets -> GPUs as contiguous rectangles of a g_y x g_x grid
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace deblur {

struct AxisFacet {
    int64_t o_lo, o_hi;   // observed [o_lo, o_hi)
    int64_t e_lo, e_hi;   // estimate [e_lo, e_hi) = [o_lo, o_hi + P - 1)
};

struct Rect {             // global estimate coordinates, half-open
    int64_t y0, y1, x0, x1;
    int64_t area() const { return (y1 - y0) * (x1 - x0); }
    bool empty() const { return y1 <= y0 || x1 <= x0; }
};

struct FacetPlan {
    int id, fy, fx, owner;
    int64_t oy0, oy1, ox0, ox1;     // observed block
    int64_t ey0, ey1, ex0, ex1;     // estimate block
    // consensus-weight ramps along each axis (global coordinates):
    //   prev band [ey0, prev_e) ramps up, next band [next_s, ey1) ramps down
    int64_t py_e, ny_s, px_e, nx_s; // prev_e (== ey0 if no prev), next_s (== ey1 if no next)
};

struct Message {          // one halo message sent per iteration
    int peer;             // destination rank
    int src_facet, dst_facet;
    Rect rect;
    int64_t bytes() const { return rect.area() * 4; }
};

struct Plan {
    int64_t ny, nx, my, mx;
    int P, Fy, Fx, O;
    int gy, gx;                      // GPU grid
    std::vector<AxisFacet> ay, ax;
    std::vector<FacetPlan> facets;   // facet-id order
    std::vector<std::string> warnings;
};

// Returns "" on success, else an error message naming the offending value.
std::string axis_plan(int64_t M, int F, int O, int P, std::vector<AxisFacet> &out);
std::string make_plan(int64_t ny, int64_t nx, int P, int Fy, int Fx, int O, int world, Plan &out);
// Rectangle shared by facets a and b (empty if not neighbours).
Rect overlap(const FacetPlan &a, const FacetPlan &b);
// Halo messages `rank` sends per iteration (ascending (dst facet, src facet)).
std::vector<Message> messages_from(const Plan &pl, int rank);
std::vector<Message> messages_to(const Plan &pl, int rank);

}  // namespace deblur
