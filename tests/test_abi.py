"""CPU checks of the boundary: the C-ABI library loads, exports every symbol
include/sforge_b200.h declares, and its host logic (grid::decompose,
neighbor topology, error texts) matches the reference (grid.hpp:44-163,
tests/test_grid.cpp:37-110).  No compute calls: there is no GPU here."""
import ctypes as C
import itertools
import os
import re

import pytest

import paper_1201_2118_b200 as sfb
from paper_1201_2118_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sforge_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = sfb.lib()
    names = declared_symbols()
    assert len(names) >= 40
    for n in names:
        assert hasattr(lib, n), n
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) == bound
    assert lib.sf_abi_version() == 2


def test_library_is_the_in_tree_build():
    assert os.path.dirname(_lib.LIB_PATH).startswith(os.path.join(ROOT, "paper_1201_2118_b200"))
    assert os.path.exists(_lib.LIB_PATH)


def _split_axis(n, p):
    base, rem = divmod(n, p)
    return [base + (1 if i < rem else 0) for i in range(p)]


def _py_decompose(ext, workers, ghost):
    # grid.hpp:92-163 restated
    best, best_area = None, None
    for px in range(1, workers + 1):
        if workers % px:
            continue
        rest = workers // px
        for py in range(1, rest + 1):
            if rest % py:
                continue
            pz = rest // py
            ok = all(p <= n and n // p > ghost for p, n in zip((px, py, pz), ext))
            if not ok:
                continue
            area = (px - 1) * ext[1] * ext[2] + (py - 1) * ext[0] * ext[2] + (pz - 1) * ext[0] * ext[1]
            if best is None or area < best_area or (area == best_area and (px > best[0] or (px == best[0] and py > best[1]))):
                best, best_area = (px, py, pz), area
    return best


def test_decompose_matches_the_reference_cases():
    d = sfb.decompose((32, 32, 32), 2, 1)
    assert d.proc_grid == (2, 1, 1)
    assert d.size(0) == (16, 32, 32) and d.lo[1] == (16, 0, 0)
    d8 = sfb.decompose((32, 32, 32), 8, 1)
    assert d8.proc_grid == (2, 2, 2) and all(d8.size(w) == (16, 16, 16) for w in range(8))
    assert sfb.decompose((64, 8, 8), 4, 1).proc_grid == (4, 1, 1)
    d1 = sfb.decompose((5, 6, 7), 1, 2)
    assert d1.lo[0] == (0, 0, 0) and d1.hi[0] == (5, 6, 7)
    assert all(d1.face_physical(0, a, s) for a in range(3) for s in range(2))
    d = sfb.decompose((8, 8, 8), 8, 1)
    assert [d.coords_of(w) for w in (1, 2, 4)] == [(0, 0, 1), (0, 1, 0), (1, 0, 0)]
    assert (d.neighbor(0, 0, 1), d.neighbor(0, 1, 1), d.neighbor(0, 2, 1), d.neighbor(0, 0, 0)) == (4, 2, 1, -1)
    dp = sfb.decompose((8, 8, 8), 2, 1, periodic=(True, True, True))
    assert dp.neighbor(0, 0, 0) == 1 and dp.neighbor(0, 0, 1) == 1 and dp.neighbor(0, 1, 0) == 0


@pytest.mark.parametrize("ext,workers,ghost", [((4, 4, 4), 8, 2), ((2, 2, 2), 16, 0), ((8, 8, 8), 0, 1), ((8, 8, 8), 1, -1)])
def test_infeasible_decompositions_raise_grid_errors(ext, workers, ghost):
    with pytest.raises(sfb.GridError):
        sfb.decompose(ext, workers, ghost)


def test_infeasible_message_is_the_reference_text():
    with pytest.raises(sfb.GridError, match=r"no feasible decomposition: 64 workers on 4x4x4 cells with ghost width 1 \(blocks must exceed the ghost width\)"):
        sfb.decompose((4, 4, 4), 64, 1)


def test_decompose_agrees_with_a_restatement_over_many_shapes():
    for ext in [(33, 17, 5), (64, 64, 64), (1024, 512, 512), (129, 129, 3), (12, 40, 7)]:
        for workers in (1, 2, 3, 4, 6, 8, 12, 16):
            for ghost in (1, 2, 3):
                best = _py_decompose(ext, workers, ghost)
                if best is None:
                    with pytest.raises(sfb.GridError):
                        sfb.decompose(ext, workers, ghost)
                    continue
                d = sfb.decompose(ext, workers, ghost)
                assert d.proc_grid == best
                sizes = [_split_axis(n, p) for n, p in zip(ext, best)]
                for w in range(workers):
                    c = d.coords_of(w)
                    lo = tuple(sum(sizes[a][: c[a]]) for a in range(3))
                    assert d.lo[w] == lo
                    assert d.size(w) == tuple(sizes[a][c[a]] for a in range(3))


def test_neighbors_are_symmetric():
    for per in itertools.product((False, True), repeat=3):
        d = sfb.decompose((24, 24, 24), 8, 1, periodic=per)
        for w in range(8):
            for a in range(3):
                for s in (0, 1):
                    nb = d.neighbor(w, a, s)
                    if nb >= 0:
                        assert d.neighbor(nb, a, 1 - s) == w
                    else:
                        assert not per[a]


def test_layout_rows_are_128_byte_aligned():
    lib = sfb.lib()
    for dims, g in [((512, 512, 512), 1), ((17, 13, 5), 2), ((129, 129, 3), 3)]:
        lay = _lib.Layout()
        d = (C.c_int64 * 3)(*dims)
        lo = (C.c_int64 * 3)(0, 0, 0)
        _lib.check(lib.sf_make_layout(d, lo, g, C.byref(lay)))
        assert lay.sx % 16 == 0 and lay.base % 16 == 0
        assert lay.sx >= dims[0] + 2 * g and lay.sy == dims[1] + 2 * g and lay.sz == dims[2] + 2 * g
        # offset(-g,-g,-g) is inside the allocation
        assert lay.base - g * lay.sy * lay.sx - g * lay.sx - g >= 0
        assert lib.sf_layout_elems(C.byref(lay)) == lay.sx * lay.sy * lay.sz


def test_cfd_constants_are_computed_as_the_reference_does():
    lib = sfb.lib()
    cfg = sfb.SolverConfig(extents=(8, 6, 4)).to_c()
    par = sfb.FluidParams(viscosity=0.02, blend=0.25).to_c()
    cc = _lib.CfdConsts()
    _lib.check(lib.sf_make_cfd_consts(C.byref(cfg), C.byref(par), C.byref(cc)))
    ix2, iy2, iz2 = 64.0, 36.0, 16.0
    act = lambda ax, ay, az: ax * ix2 + ay * iy2 + az * iz2  # noqa: E731
    want = [act(2.0, 2.0, 2.0) / act(2.0 if bx else 1.0, 2.0 if by else 1.0, 2.0 if bz else 1.0)
            for bx in (0, 1) for by in (0, 1) for bz in (0, 1)]
    assert list(cc.bscale) == want
    assert cc.bscale[7] == 1.0
    assert (cc.nxm1, cc.nym1, cc.nzm1) == (7, 5, 3)


def test_no_gpu_here_fails_loudly_not_silently():
    if sfb.lib().sf_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(sfb.SfError) as e:
        sfb.Simulation(sfb.SolverConfig(extents=(8, 8, 8)), sfb.FluidParams())
    assert e.value.kind == "cuda"


def test_cpp_header_compiles_against_the_library(tmp_path):
    """The C++ face (include/sforge_b200.hpp) builds and links against the
    in-tree library; without a GPU it reports the CUDA failure as an exception."""
    import subprocess
    exe = tmp_path / "cavity_cpp"
    lib_dir = os.path.dirname(_lib.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "cavity_cpp.cpp"), "-L" + lib_dir, "-lsfb200",
                        "-Wl,-rpath," + lib_dir, "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    if sfb.lib().sf_device_count() == 0:
        out = subprocess.run([str(exe), "8", "1"], capture_output=True, text=True)
        assert out.returncode == 1 and "error:" in out.stdout


def test_library_stamp_is_the_hash_of_its_sources():
    # freshness by content, not file times: a copied tree keeps its prebuilt
    # library, and concurrent importers see one consistent answer
    from paper_1201_2118_b200 import build
    sfb.lib()  # builds (and stamps) the library if it is missing or stale
    assert os.path.exists(build.STAMP)
    assert open(build.STAMP).read().strip() == build.source_hash()
    assert not build._stale()


def test_bench_reports_ncu_traffic_only_for_its_workload():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import json
    cap = json.load(open(os.path.join(ROOT, "profiles", "ncu_sweep2.json")))
    t, src = bench.ncu_traffic("sweep2", cap["algo_bytes_per_launch"])
    assert t == cap["dram_bytes_per_launch"] and src["captured_from"] == cap["captured_from"]
    assert "not_applicable" not in src
    t, src = bench.ncu_traffic("sweep2", 8 * cap["algo_bytes_per_launch"])  # e.g. the 1024^3 pass
    assert t is None and "not_applicable" in src
