"""Pins the CPU oracles (test infrastructure) before anything is checked
against them: the plain-C restatement (oracle/sf_oracle.c) against the golden
checksums of SURVEY.md Appendix A and bitwise against the reference compiled
in place (oracle/_ref/libsfref.so)."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import Case, Oracle, available, cavity_case

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def test_port_reproduces_the_64_cube_golden_checksum_after_one_step():
    o = Oracle(cavity_case(64, symmetry_z=False), "port")
    o.init_cavity()
    dt, sweeps, res = o.step()
    assert o.checksum() == GOLDEN["cavity64"]["checksums"]["1"] == "1b07d1f577d4bad0"
    assert dt == 0.0020345052083333335
    assert sweeps == 500
    assert [dt, sweeps, res] == GOLDEN["cavity64"]["stats"][0]


def test_port_reproduces_the_golden_after_ten_steps():
    o = Oracle(cavity_case(64, symmetry_z=False), "port")
    o.init_cavity()
    dts, sw, res = o.advance(10)
    assert o.checksum() == "32b900f8b9e72ed2"
    assert [[float(a), int(b), float(c)] for a, b, c in zip(dts, sw, res)] == GOLDEN["cavity64"]["stats"]


def test_port_reproduces_the_quasi2d_and_ghost_width_goldens():
    o = Oracle(cavity_case((33, 33, 3), sigma=0.8), "port")
    o.init_cavity()
    o.advance(20)
    assert o.checksum() == GOLDEN["quasi2d_33"]["checksums"]["20"]
    o = Oracle(cavity_case(24, symmetry_z=False, ghost=2), "port")
    o.init_cavity()
    o.advance(3)
    assert o.checksum() == GOLDEN["cavity24_g2"]["checksums"]["3"]


def _random_fields(shape, seed):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1.0, 1.0, size=shape[::-1]) for _ in range(3)]


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("ghost", [1, 2])
def test_port_matches_the_reference_bitwise_on_random_fields(ref_available, periodic, ghost):
    # the shape of tests/test_cfd.cpp:275-325: odd extents, capped sweeps
    ext = (17, 13, 5)
    vx, vy, vz = _random_fields(ext, 13)
    outs = []
    for kind in ("ref", "port"):
        c = Case(extents=ext, periodic=(periodic,) * 3, tolerance=1e-12, max_sweeps=40,
                 viscosity=0.05, lid_speed=0.0 if periodic else 1.0, ghost=ghost)
        o = Oracle(c, kind)
        o.scatter("vx", vx)
        o.scatter("vy", vy)
        o.scatter("vz", vz)
        o.invalidate_all_ghosts()
        stats = o.advance(2)
        outs.append(([o.gather(f) for f in ("vx", "vy", "vz", "p", "divu")], [list(s) for s in stats]))
    (a, sa), (b, sb) = outs
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
    assert sa == sb


def test_port_matches_reference_ghosts_after_a_refresh(ref_available):
    ext = (9, 7, 6)
    for kind_bc in (dict(symmetry_z=True), dict(symmetry_z=False), dict(periodic=(True, False, True))):
        arrs = {}
        for kind in ("ref", "port"):
            o = Oracle(Case(extents=ext, lid_speed=0.7, ghost=2, **kind_bc), kind)
            for i, f in enumerate(("vx", "vy", "vz", "p", "divu")):
                o.scatter(f, np.random.default_rng(i).standard_normal(ext[::-1]))
            o.refresh(["vx", "vy", "vz", "p", "divu"])
            arrs[kind] = [o.local_front(f) for f in ("vx", "vy", "vz", "p", "divu")]
        for x, y in zip(arrs["ref"], arrs["port"]):
            assert np.array_equal(x, y)


def test_reference_golden_fixture_is_reproducible(ref_available):
    o = Oracle(cavity_case(24, symmetry_z=False, ghost=3), "ref")
    o.init_cavity()
    o.advance(2)
    assert o.checksum() == GOLDEN["cavity24_g3_w1"]["checksums"]["2"]


def _taylor_green_run(backend, n, workers=1, T=0.5):
    # acceptance check 6's loop (tests/acceptance/acceptance_main.cpp:416-440)
    c = Case(extents=(n, n, 2), periodic=(True, True, True), tolerance=1e-8, max_sweeps=20000, viscosity=0.01,
             lid_speed=0.0, workers=workers)
    o = Oracle(c, backend)
    o.init_taylor_green()
    t, steps, sweeps = 0.0, 0, 0
    while t < T:
        dt = min(o.compute_dt(), T - t)
        o.provisional(dt)
        sw, _ = o.pressure_iteration(dt)
        o.refresh(["p"])
        t += dt
        steps += 1
        sweeps += sw
    return o.taylor_green_error(T), steps, sweeps


def test_port_taylor_green_error_matches_the_reference(ref_available):
    # cfd.hpp:367-401 restated in C: bitwise on one worker, at the start and
    # after the vortex decays to T = 0.5
    for T in (0.0, 0.5):
        assert _taylor_green_run("port", 16, T=T) == _taylor_green_run("ref", 16, T=T)


def test_taylor_green_order_golden_is_the_reference_check_6(ref_available):
    # the acceptance-6 fixture (2 workers, 32^2 and 64^2): error falls >= 3.6x
    g = GOLDEN["taylor_green_order"]
    assert list(_taylor_green_run("ref", 32, workers=2)) == g["32"]
    assert g["32"][0] / g["64"][0] >= 3.6


def test_sfg1_format_round_trips_the_reference_cli_dumps(tmp_path):
    # grid::write_sfg1 / read_sfg1 (io.hpp:66-101): files written by the
    # reference's `sforge cavity` read back and rewrite byte for byte
    import io
    import subprocess

    from paper_1201_2118_b200 import GridError
    from paper_1201_2118_b200.cavity import read_sfg1, write_sfg1
    cli = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "sforge")
    if not os.path.exists(cli):
        pytest.skip("oracle/_ref/sforge not built")
    (tmp_path / "c.cfg").write_text("nx = 9\nny = 7\nnz = 3\nmax_steps = 3\nsteady_tol = 1e-30\nfields_out = f\n"
                                    "profiles_out = p.csv\nresiduals_out = r.csv\n")
    # (exits 1: "not steady after 3 steps"; the dumps are written first)
    subprocess.run([cli, "cavity", "--config", "c.cfg"], cwd=tmp_path, capture_output=True, timeout=300)
    for name in ("vx", "vy", "vz", "p"):
        blob = (tmp_path / "f" / (name + ".sfg1")).read_bytes()
        ext, data = read_sfg1(io.BytesIO(blob))
        assert ext == (9, 7, 3) and data.shape == (3, 7, 9)
        out = io.BytesIO()
        write_sfg1(out, ext, data)
        assert out.getvalue() == blob
    with pytest.raises(GridError, match="not an SFG1 stream"):
        read_sfg1(io.BytesIO(b"XXXX"))
    with pytest.raises(GridError, match="truncated payload"):
        read_sfg1(io.BytesIO(blob[:-8]))
    with pytest.raises(GridError, match="does not match extents"):
        write_sfg1(io.BytesIO(), (2, 2, 2), np.zeros(7))
