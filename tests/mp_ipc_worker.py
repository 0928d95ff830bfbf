"""One rank of a multi-process run of the cross-process data plane (launched by
tests/test_gpu_multiproc.py through torch.distributed.run).

Every rank owns one grid component of grid::decompose(dom, world, ghost)
(grid.hpp:92-163) and exchanges ghosts with its peers through the CUDA-IPC
transport (include/sforge_b200.h sf_sim_create_ipc): pack tasks, the posting
order of the messages, pulls out of the peers' send buffers, unpack tasks,
the max-allreduce of the residuals and the cross-rank loop decision
(CTL_FINISH_FUSED / CTL_FINISH_PASS), and -- for the temporal pass -- the
direct stores into the peers' ghost shells.  All ranks may share one GPU: no
kernel waits on another rank's kernel, the host orders them (gloo barriers).

Rank 0 compares every variant with the reference (oracle/_ref) run with the
same worker count: per-step (dt, sweeps, residual) and the FNV checksum of the
gathered fields, bitwise.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1201_2118_b200 as sfb  # noqa: E402

VARIANTS = {  # name: (fused, direct exchange mode)
    "temporal-direct-fused": (1, 1),     # boundary cells of the pass store into the peers' ghosts
    "temporal-direct-launch": (1, 2),    # one launch of direct stores after each pass
    "temporal-phases-overlapped": (1, 0),  # pack / pull / unpack phases beside the interior tiles
    "single-half-sweep": (3, 1),
    "unfused": (0, 1),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ext", type=int, nargs=3, required=True)
    ap.add_argument("--ghost", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--max-sweeps", type=int, default=41)
    ap.add_argument("--tolerance", type=float, default=1e-4)
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--periodic", type=int, nargs=3, default=[0, 0, 0])
    ap.add_argument("--one-device", action="store_true", help="every rank on cuda:0")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import datetime
    dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=300))
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = 0 if a.one_device else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    per = tuple(bool(x) for x in a.periodic)
    cfg = sfb.SolverConfig(extents=tuple(a.ext), periodic=per, reynolds=100.0, omega=1.9525,
                           tolerance=a.tolerance, max_sweeps=a.max_sweeps, symmetry_z=False)
    results = {}
    for name in a.variants.split(","):
        fused, direct = VARIANTS[name]
        sim = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), ghost=a.ghost, device=dev, fused=fused, rank=rank,
                             world=world, transport="ipc")
        sim.set_direct_exchange(direct)
        print(f"rank {rank}: variant {name}", flush=True)
        sim.init_cavity()
        sim.set_kernel_timing(True)
        stats = [sim.step() for _ in range(a.steps)]
        csum = sim.checksum()  # collective: grid::gather over the ranks
        used_direct = sim.direct_exchange if fused == 1 else 0
        results[name] = {"stats": [[s.dt, s.sweeps, s.residual] for s in stats], "checksum": csum,
                         "passes": sim.kernel_timing("sweep2")[1], "half_sweeps": sim.kernel_timing("sweep_div")[1],
                         "interior": sim.kernel_timing("sweep2i")[1],
                         "direct": used_direct, "block": list(sim.block_shape())}
        dist.barrier()
        sim.close()
        dist.barrier()
    if rank == 0:
        from oracle.oracle import Oracle, cavity_case
        c = cavity_case(tuple(a.ext), periodic=per, symmetry_z=False, omega=1.9525, tolerance=a.tolerance,
                        max_sweeps=a.max_sweeps, ghost=a.ghost, workers=world)
        o = Oracle(c, "ref")
        o.init_cavity()
        so = o.advance(a.steps)
        want = [[float(x), int(y), float(z)] for x, y, z in zip(*so)]
        out = {"world": world, "reference": {"stats": want, "checksum": o.checksum()}, "variants": results}
        for r in results.values():
            r["ok"] = r["stats"] == want and r["checksum"] == out["reference"]["checksum"]
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
