"""`python -m paper_1201_2118_b200` against the reference's own CLI
(oracle/_ref/sforge, built from proj/tools/sforge.cpp): the same stdout,
files and exit status for `gen` and `validate` (CPU), and for `cavity` on the
GPU (tests/test_gpu_parity.py)."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "sforge")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def run_both(args, tmp_path, files=()):
    """Runs both CLIs in sibling directories holding copies of `files`;
    returns ((rc, stdout, stderr) mine, (rc, stdout, stderr) reference)."""
    if not os.path.exists(REF_CLI):
        pytest.skip("oracle/_ref/sforge not built")
    out = []
    for name, cmd in (("mine", [sys.executable, "-m", "paper_1201_2118_b200"]), ("ref", [REF_CLI])):
        d = tmp_path / name
        d.mkdir()
        for src, dst in files:
            shutil.copy(src, d / dst)
        env = dict(os.environ, PYTHONPATH=ROOT)
        p = subprocess.run(cmd + list(args), cwd=d, capture_output=True, text=True, timeout=300, env=env)
        out.append((p.returncode, p.stdout, p.stderr))
    return out


CCL = """CCTK_CUDA_KERNEL SMOOTH TYPE=3DBLOCK STENCIL="1,1,1,1,1,1" TILE="8,4,4"
{
  CCTK_CUDA_KERNEL_VARIABLE CACHED=YES INTENT=IN { src } "SOURCE"
  CCTK_CUDA_KERNEL_VARIABLE INTENT=OUT { dst } "RESULT"
  CCTK_CUDA_KERNEL_PARAMETER { weight } "W"
}
CCTK_CUDA_KERNEL SHIFT TYPE=3DBLOCK STENCIL="0,1,0,0,0,0" TILE="2,2,2"
{
  CCTK_CUDA_KERNEL_VARIABLE INTENT=SEPARATEINOUT { v } "V"
}
"""


def test_gen_writes_the_reference_headers_and_manifest(tmp_path):
    src = tmp_path / "k.ccl"
    src.write_text(CCL)
    mine, ref = run_both(["gen", "k.ccl", "-o", "out"], tmp_path, [(src, "k.ccl")])
    assert mine == ref and mine[0] == 0
    for n in sorted(os.listdir(tmp_path / "ref" / "out")):
        assert (tmp_path / "mine" / "out" / n).read_bytes() == (tmp_path / "ref" / "out" / n).read_bytes(), n


@pytest.mark.parametrize("args", [[], ["gen"], ["gen", "k.ccl"], ["gen", "-x"], ["frobnicate"],
                                  ["gen", "missing.ccl", "-o", "o"], ["validate", "--tol", "abc"],
                                  ["cavity"], ["cavity", "--workers", "0"], ["cavity", "--config", "none.cfg"],
                                  ["bench"], ["bench", "--workers", "1,0"], ["bench", "--modes", "fast"],
                                  ["bench", "--steps", "0"], ["help"]])
def test_usage_and_input_errors_match(tmp_path, args):
    mine, ref = run_both(args, tmp_path)
    assert mine == ref


def test_gen_reports_descriptor_errors_like_the_reference(tmp_path):
    src = tmp_path / "bad.ccl"
    src.write_text(CCL.replace('TILE="2,2,2"', 'TILE="2,0,2"'))
    mine, ref = run_both(["gen", "bad.ccl", "-o", "out"], tmp_path, [(src, "bad.ccl")])
    assert mine == ref and mine[0] == 1


@pytest.mark.parametrize("tol", ["0.03", "0.001"])
def test_validate_prints_the_reference_deviation_table(tmp_path, tol):
    files = [(os.path.join(GOLDEN, "re100_profiles.csv"), "p.csv"), (os.path.join(GOLDEN, "ghia_re100.csv"), "g.csv")]
    mine, ref = run_both(["validate", "--profiles", "p.csv", "--reference", "g.csv", "--tol", tol], tmp_path, files)
    assert mine == ref
    assert mine[0] == (0 if tol == "0.03" else 1)


@pytest.mark.parametrize("bad", ["y,u\n0,1\n", "0,1\n", "y,u\n0,1\n0,2\nx,v\n0,1\n1,2\n", "y,u\n0;1\n",
                                 "y,u\n0,1x\n", "y,u\nzero,1\n"])
def test_validate_rejects_malformed_profiles_like_the_reference(tmp_path, bad):
    src = tmp_path / "bad.csv"
    src.write_text(bad)
    files = [(src, "b.csv"), (os.path.join(GOLDEN, "ghia_re100.csv"), "g.csv")]
    mine, ref = run_both(["validate", "--profiles", "b.csv", "--reference", "g.csv", "--tol", "1"], tmp_path, files)
    assert mine == ref and mine[0] == 1
