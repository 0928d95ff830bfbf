"""Host / device transfers of the public API (io.hpp:25-65 semantics): stream
ordering against torch's work, and the buffer checks of the raw-pointer paths."""
import numpy as np
import pytest

import paper_1201_2118_b200 as sfb

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _sim(ext=(40, 24, 20)):
    cfg = sfb.SolverConfig(extents=ext, symmetry_z=False)
    s = sfb.Simulation(cfg, sfb.cavity_fluid(cfg))
    s.init_cavity()
    return s


def test_device_scatter_and_gather_are_ordered_with_torch_streams():
    s = _sim()
    n = 40 * 24 * 20
    for seed in range(3):
        # the input is produced by queued torch work, consumed at once, and the
        # temporary of .contiguous() is dropped right after the call
        base = torch.randn(20, 24, 40 * 2, dtype=torch.float64, device="cuda", generator=torch.Generator(
            device="cuda").manual_seed(seed))
        for _ in range(20):
            base = base * 1.0000001 + 1e-9  # keep torch's stream busy
        s.scatter("vx", base[:, :, ::2])  # non-contiguous view: copied to a temporary
        out = torch.full((n,), np.nan, dtype=torch.float64, device="cuda")
        s.gather("vx", out=out)
        got = (out * 1.0).cpu().numpy()  # torch work right after the gather sees its values
        assert np.array_equal(got, base[:, :, ::2].contiguous().reshape(-1).cpu().numpy())
        assert np.array_equal(s.gather("vx").reshape(-1), got)


def test_raw_pointer_paths_reject_wrong_buffers():
    s = _sim()
    n = 40 * 24 * 20
    with pytest.raises(ValueError, match="float64"):
        s.gather("vx", out=torch.empty(n, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError, match="float64"):
        s.gather("vx", out=np.empty(n, dtype=np.float32))
    with pytest.raises(ValueError, match="float64"):
        s.gather_block("vx", out=np.empty(n, dtype=np.int64))
    with pytest.raises(ValueError, match="pinned"):
        s.gather_block("vx", out=torch.empty(n, dtype=torch.float64), wait=False)
    with pytest.raises(ValueError, match="pinned"):
        s.scatter_block("vx", torch.zeros(n, dtype=torch.float64), wait=False)
    with pytest.raises(ValueError, match="pinned"):
        s.stage_block("vx", torch.zeros(n, dtype=torch.float64))
    with pytest.raises(ValueError, match="contiguous"):
        s.scatter_block("vx", torch.zeros(2 * n, dtype=torch.float64).pin_memory()[::2])
    # an int64 tensor is converted by value, never read as raw double bits
    s.scatter("vy", torch.arange(n, dtype=torch.int64))
    assert np.array_equal(s.gather("vy").reshape(-1), np.arange(n, dtype=np.float64))


def test_async_buffers_stay_referenced_until_synchronize():
    s = _sim()
    n = 40 * 24 * 20
    want = np.random.default_rng(5).standard_normal(n)
    for _ in range(4):  # temporaries: the simulation keeps them alive until synchronize()
        s.scatter_block("vz", torch.from_numpy(want.copy()).pin_memory(), wait=False)
        s.gather_block("vz", out=torch.empty(n, dtype=torch.float64).pin_memory(), wait=False)
    s.synchronize()
    assert np.array_equal(s.gather("vz").reshape(-1), want)


def test_device_gather_then_block_download_sees_the_gathered_state():
    # a device scatter followed by a synchronous block download: the download
    # must wait for the scatter's kernel (compute epoch bumped by the launch)
    s = _sim()
    n = 40 * 24 * 20
    for seed in range(5):
        src = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator(
            device="cuda").manual_seed(seed))
        s.scatter("p", src)
        blk = s.gather_block("p")
        assert np.array_equal(blk.reshape(-1), src.cpu().numpy())
