"""The C++ executor drop-in (include/sforge_b200.hpp, namespace
sforge_b200::exec) against the reference executor running the SAME point
functors (SF_POINT_FUNCTION): tests/cpp/executor_functors.cpp is compiled once
against the reference headers (oracle/_ref/executor_functors_ref, built by
oracle/Makefile) and once against this library; every gathered field is
compared bitwise and every reduce result (max bitwise, sums to rounding).
Cases mirror the reference's tests/test_executor.cpp: identity, tiling /
caching / worker-count transparency (periodic), an asymmetric halo with
separate in/out, parameters by slot and regions, global indices, and moving
walls / symmetry / outflow under staggered fields through a schedule with
refresh, kernel and reductions in plain and overlap mode."""
import os
import struct
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_EXE = os.path.join(ROOT, "oracle", "_ref", "executor_functors_ref")


def read_records(path):
    out = {}
    with open(path, "rb") as f:
        data = f.read()
    at = 0
    while at < len(data):
        (nl,) = struct.unpack_from("i", data, at)
        at += 4
        name = data[at:at + nl].decode()
        at += nl
        (n,) = struct.unpack_from("q", data, at)
        at += 8
        out[name] = np.frombuffer(data, dtype=np.float64, count=n, offset=at).copy()
        at += 8 * n
    return out


def test_same_point_functors_match_the_reference_executor(tmp_path):
    if not os.path.exists(REF_EXE):
        pytest.skip("oracle/_ref/executor_functors_ref not built (make -C oracle ref)")
    lib_dir = os.path.join(ROOT, "paper_1201_2118_b200", "_lib")
    exe = tmp_path / "executor_functors"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "executor_functors.cpp"), "-L" + lib_dir, "-lsfb200",
                        "-Wl,-rpath," + lib_dir, "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    ours, ref = tmp_path / "ours.bin", tmp_path / "ref.bin"
    for cmd, out in ((str(exe), ours), (REF_EXE, ref)):
        p = subprocess.run([cmd, str(out)], capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, (cmd, p.stdout, p.stderr)
    a, b = read_records(ours), read_records(ref)
    assert a.keys() == b.keys() and len(a) >= 20
    for k in a:
        if "~" in k:  # sums: the device folds in another order (equal to rounding)
            assert np.allclose(a[k], b[k], rtol=1e-12, atol=1e-12), k
        else:
            assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k
