"""Time the multi-GPU code path in a one-process NCCL world against the single-GPU evolve.

    python tools/time_sharded.py [--n 16384] [--steps 100]

ShardedSolver(force_split=True) runs exactly what each rank of a multi-GPU job runs (pair
split, NCCL reduce-scatter, stage finish, NCCL all-gather) with world = 1, so the difference
to device.evolve is the orchestration overhead of the sharded path.
"""

from __future__ import annotations

import argparse
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--path", default="auto")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1510_03816_b200 as gs
    from paper_1510_03816_b200 import configs, device, sharded

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    gs.set_path(a.path)
    w = configs.c2(a.n)
    spec = gs.SystemSpec(kernel=gs.KernelSpec(alpha=w.alpha))
    q = torch.from_numpy(w.q).cuda()
    p = torch.from_numpy(w.p).cuda()
    solver = sharded.ShardedSolver(spec, force_split=True)

    def t(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    ts = t(lambda: solver.evolve(q, p, 1.0, a.steps))
    td = t(lambda: device.evolve(spec, q, p, 1.0, a.steps))
    qa, pa = solver.evolve(q, p, 1.0, a.steps)
    qb, pb, _ = device.evolve(spec, q, p, 1.0, a.steps)
    err = float((qa - qb).abs().max() / qb.abs().max())
    print(f"n={a.n} steps={a.steps} sharded(world1) {ts*1e3:.2f} ms  single {td*1e3:.2f} ms  "
          f"per-stage overhead {(ts-td)/(4*a.steps)*1e6:.1f} us  rel diff {err:.2e}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
