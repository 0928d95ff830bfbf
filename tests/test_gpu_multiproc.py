"""The cross-process data plane with real peers (several processes, one GPU).

NCCL refuses two ranks on one device, so these runs use the library's
CUDA-IPC transport (sf_sim_create_ipc): each rank is its own process with its
own CUDA context, maps its peers' device buffers, and moves every ghost
message through them -- pack tasks (k_tasks type 2), the per-peer posting
order, device copies out of the peers' send buffers, unpack tasks (type 3),
the residual max-allreduce and the cross-rank loop decisions
(CTL_FINISH_FUSED / CTL_FINISH_PASS), and for the temporal pass the direct
stores into the peers' ghost shells -- fused into the pass's epilogue, or
as one separate launch (k_tasks type 4) -- or the overlapped three-phase
exchange.  No kernel waits on another rank's kernel (the host orders them
with gloo barriers), so co-scheduling the ranks on one GPU is safe.

Each run is compared bitwise with the reference at the same worker count
(exchange.hpp:98-224; tests/test_grid.cpp:195-252 is the reference's own
multi-worker exchange test).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, ext, tmp_path, extra=()):
    out = tmp_path / f"mp{world}.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(HERE, "mp_ipc_worker.py"),
           "--one-device", "--ext", *map(str, ext), "--out", str(out), *extra]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    return json.loads(out.read_text())


@pytest.mark.parametrize("world,ext", [(2, (136, 40, 24)), (4, (140, 84, 30))])
def test_ranks_in_separate_processes_match_the_reference(ref_available, world, ext, tmp_path):
    res = _run(world, ext, tmp_path)
    assert res["world"] == world
    for name, v in res["variants"].items():
        assert v["ok"], (name, v, res["reference"])
    v = res["variants"]
    assert v["temporal-direct-fused"]["direct"] == 1 and v["temporal-direct-fused"]["passes"] > 0
    # with the exchange fused into the slabs' stores, every pass runs the
    # interior form (k_sweep2i) beside the REMOTE slab launches
    assert v["temporal-direct-fused"]["interior"] == v["temporal-direct-fused"]["passes"]
    assert v["temporal-phases-overlapped"]["interior"] == 0
    assert v["temporal-direct-launch"]["direct"] == 2 and v["temporal-direct-launch"]["passes"] > 0
    assert v["temporal-phases-overlapped"]["direct"] == 0 and v["temporal-phases-overlapped"]["passes"] > 0
    assert v["single-half-sweep"]["passes"] == 0 and v["single-half-sweep"]["half_sweeps"] > 0
    # blocks large enough that the overlapped variant has interior tiles
    assert v["temporal-phases-overlapped"]["block"][0] >= 66


def test_odd_stop_parities_and_periodic_wrap_across_processes(ref_available, tmp_path):
    # odd sweep caps (a pass stops after its first sweep on every rank: the
    # redo kernel), uneven blocks, and a periodic x axis split over three
    # ranks (processor faces through the wrap, odd global extent)
    res = _run(3, (99, 37, 21), tmp_path, ["--max-sweeps", "9", "--tolerance", "1e-30", "--steps", "3",
                                           "--periodic", "1", "0", "0"])
    for name, v in res["variants"].items():
        assert v["ok"], (name, v, res["reference"])
