"""N > 1 path on CPU: world-size-2 (and 4) gloo ranks emulate the distributed
iteration with libdeblur's own plan (facet -> rank map, halo messages from
deblur_plan_messages) and the oracle's arithmetic, exchanging v = 2x+ - u bands
over gloo exactly as the NCCL path does on GPUs.  The result must equal the
single-process oracle iteration (same ascending-facet-id consensus order), and
the message lists must be pairwise consistent across ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import from_problem
from paper_1705_06603_b200 import deblur as D


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def problem():
    return synth.make_config(2, n=256, facets=(2, 2), overlap=32)


def worker(rank, world, port, iters, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pb = problem()
        params, keep = D.problem_params(pb, rank=rank, world=world, nccl_id_bytes=b"\0" * 128)
        boxes, owner = D.plan_facets(params)
        sends = D.plan_messages(params, rank)
        recvs = np.concatenate([D.plan_messages(params, r) for r in range(world) if r != rank] or
                               [np.zeros((0, 8), np.int64)])
        recvs = recvs[recvs[:, 0] == rank] if len(recvs) else recvs
        # pairwise consistency: what I receive is what my peers send me
        counts = torch.tensor([len(sends)], dtype=torch.int64)
        allc = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, counts)
        orc = from_problem(pb)
        mine = [f for f in range(len(boxes)) if owner[f] == rank]
        for _ in range(iters):
            # Local-Solver on my facets only
            for f in mine:
                orc.x[f] = orc.local_prox(f, orc.x[f], orc.u[f])
            v = {f: 2 * orc.x[f] - orc.u[f] for f in mine}
            # halo exchange over gloo, per message rectangle (global estimate coords)
            reqs = []
            for m in sends:
                peer, s, d_, y0, y1, x0, x1, _ = (int(t) for t in m)
                ey0, ex0 = boxes[s][4], boxes[s][6]
                buf = torch.from_numpy(np.ascontiguousarray(v[s][y0 - ey0:y1 - ey0, x0 - ex0:x1 - ex0]))
                reqs.append(dist.isend(buf, peer))
            got = {}
            for m in recvs:
                src_rank, s, d_, y0, y1, x0, x1, nbytes = (int(t) for t in m)
                src = int(owner[s])
                buf = torch.zeros((y1 - y0, x1 - x0), dtype=torch.float64)
                dist.recv(buf, src)
                got[(s, d_)] = (buf.numpy(), y0, x0)
            for r in reqs:
                r.wait()
            # consensus (Lemma 1) for my facets, contributions in ascending facet id
            for f in mine:
                fey0, fey1, fex0, fex1 = boxes[f][4:8]
                num = np.zeros((fey1 - fey0, fex1 - fex0))
                den = np.zeros_like(num)
                for g in range(len(boxes)):
                    gy0, gy1, gx0, gx1 = boxes[g][4:8]
                    y0, y1, x0, x1 = max(fey0, gy0), min(fey1, gy1), max(fex0, gx0), min(fex1, gx1)
                    if y0 >= y1 or x0 >= x1:
                        continue
                    om = orc.omegas[g][y0 - gy0:y1 - gy0, x0 - gx0:x1 - gx0]
                    if g in v:
                        vg = v[g][y0 - gy0:y1 - gy0, x0 - gx0:x1 - gx0]
                    else:
                        arr, ry0, rx0 = got[(g, f)]
                        vg = arr[y0 - ry0:y1 - ry0, x0 - rx0:x1 - rx0]
                    sl = (slice(y0 - fey0, y1 - fey0), slice(x0 - fex0, x1 - fex0))
                    num[sl] = num[sl] + om * vg
                    den[sl] = den[sl] + om
                orc.u[f] = orc.u[f] + orc.prm.rho * (num / den - orc.x[f])
        q.put((rank, {f: (orc.x[f], orc.u[f]) for f in mine}, [int(c) for c in allc],
               sum(len(D.plan_messages(params, r)) for r in range(world))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_iteration_matches_single_process(world):
    iters = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = from_problem(problem())
    ref.iterate(iters)
    seen = set()
    for rank, facets, counts, total_msgs in res:
        assert sum(counts) == total_msgs
        for f, (x, u) in facets.items():
            seen.add(f)
            np.testing.assert_allclose(x, ref.x[f], rtol=0, atol=1e-13)
            np.testing.assert_allclose(u, ref.u[f], rtol=0, atol=1e-13)
    assert seen == set(range(4))
