"""The descriptor front end (paper_1201_2118_b200/descriptor.py) against the
reference's own (descriptor.hpp, codegen.hpp, compiled in place into
oracle/_ref/libsfref.so): structure, canonical rendering, validation errors,
rendered headers and the plans manifest, on the reference's test inputs
(tests/test_descriptor.cpp, test_codegen.cpp, acceptance check 1) and on
randomly mutated descriptor files. CPU only."""
import os
import random

import pytest

from oracle.oracle import ref_ccl
from paper_1201_2118_b200 import descriptor as D

# The three kernels of the CFD step in descriptor form (the contract of
# cfd.hpp:106-163 / kernels/cfd.ccl), written out here in this repo's layout.
CFD_CCL = """# kernels of the projection step
CCTK_CUDA_KERNEL UPDATE_VELOCITY TYPE=3DBLOCK STENCIL="1,1,1,1,1,1" TILE="16,16,16"
{
  CCTK_CUDA_KERNEL_VARIABLE CACHED=YES INTENT=SEPARATEINOUT { vx, vy, vz } "VELOCITY"
  CCTK_CUDA_KERNEL_VARIABLE CACHED=YES INTENT=IN { p } "PRESSURE"
  CCTK_CUDA_KERNEL_PARAMETER { density } "DENSITY"
}
CCTK_CUDA_KERNEL DIVERGENCE TYPE=3DBLOCK STENCIL="1,0,1,0,1,0" TILE="16,16,16"
{
  CCTK_CUDA_KERNEL_VARIABLE CACHED=NO INTENT=IN { vx, vy, vz } "VELOCITY"
  CCTK_CUDA_KERNEL_VARIABLE CACHED=NO INTENT=OUT { divu } "DIVERGENCE"
}
CCTK_CUDA_KERNEL PRESSURE_SWEEP TYPE=3DBLOCK STENCIL="0,1,0,1,0,1" TILE="16,16,16"
{
  CCTK_CUDA_KERNEL_VARIABLE CACHED=NO INTENT=IN { divu } "DIVERGENCE"
  CCTK_CUDA_KERNEL_VARIABLE CACHED=NO INTENT=INOUT { p, vx, vy, vz } "CORRECTED"
  CCTK_CUDA_KERNEL_PARAMETER { beta, color } "SWEEP"
}
"""
CFD_FIELDS = ["vx", "vy", "vz", "p", "divu"]


def mine(text, fields=None, directory=None):
    """This module's result in ref_ccl's (rc, text) form."""
    try:
        raw = D.parse_descriptors(text)
        if fields is None:
            return 0, D.render(raw)
        ks = D.validate_all(raw, fields)
        if directory is not None:
            D.write_generated(ks, directory)
        return 0, "".join(D.render_header(k)[0] for k in ks)
    except D.ParseError as e:
        return 1, str(e)
    except D.DescriptorError as e:
        return 2, str(e)


def test_golden_kernel_structure_round_trip_and_render_fixed_point():
    # acceptance check 1 (acceptance_main.cpp:143-176) on UPDATE_VELOCITY
    ks = D.parse_descriptors(CFD_CCL)
    k = ks[0]
    assert [x.name for x in ks] == ["UPDATE_VELOCITY", "DIVERGENCE", "PRESSURE_SWEEP"]
    assert k.attrs == [("TYPE", D.AttrValue("3DBLOCK", False)), ("STENCIL", D.AttrValue("1,1,1,1,1,1", True)),
                       ("TILE", D.AttrValue("16,16,16", True))]
    g0, g1, g2 = k.groups
    assert not g0.parameter and g0.names == ["vx", "vy", "vz"] and g0.description == "VELOCITY"
    assert g0.attrs == [("CACHED", D.AttrValue("YES")), ("INTENT", D.AttrValue("SEPARATEINOUT"))]
    assert not g1.parameter and g1.names == ["p"] and g1.description == "PRESSURE"
    assert g2.parameter and g2.names == ["density"] and g2.description == "DENSITY"
    canonical = D.render(ks)
    again = D.parse_descriptors(canonical)
    assert again == ks and D.render(again) == canonical


def test_plans_of_the_cfd_kernels():
    plans = D.load_plans(CFD_CCL, CFD_FIELDS)
    uv = plans["UPDATE_VELOCITY"]
    assert uv.tile == (16, 16, 16) and uv.halo == (1, 1, 1, 1, 1, 1)
    assert uv.bindings == (("vx", "SEPARATEINOUT", True), ("vy", "SEPARATEINOUT", True),
                           ("vz", "SEPARATEINOUT", True), ("p", "IN", True))
    assert uv.parameters == ("density",)
    assert plans["DIVERGENCE"].halo == (1, 0, 1, 0, 1, 0)
    assert plans["PRESSURE_SWEEP"].parameters == ("beta", "color")


def test_the_reference_renders_and_generates_the_same(ref_available, tmp_path):
    assert mine(CFD_CCL) == ref_ccl(CFD_CCL)
    a, b = tmp_path / "mine", tmp_path / "ref"
    assert mine(CFD_CCL, CFD_FIELDS, str(a)) == ref_ccl(CFD_CCL, CFD_FIELDS, str(b))
    names = sorted(os.listdir(b))
    assert sorted(os.listdir(a)) == names == ["DIVERGENCE.h.generated", "PRESSURE_SWEEP.h.generated",
                                               "UPDATE_VELOCITY.h.generated", "plans.txt"]
    for n in names:
        assert (a / n).read_bytes() == (b / n).read_bytes(), n


# inputs of the reference's own tests (test_descriptor.cpp:72-215, test_codegen.cpp)
_K = 'CCTK_CUDA_KERNEL K TYPE=3DBLOCK STENCIL="0,0,0,0,0,0" TILE="4,4,4" '
CASES = [
    "",
    "# only a comment\n\n",
    "CCTK_CUDA_KERNEL K TYPE=3DBLOCK\n{\n  CCTK_CUDA_KERNEL_VARIABLE { p } \"X\"\n",
    "CCTK_CUDA_KERNEL\n",
    "junk\n",
    "CCTK_CUDA_KERNEL K { } trailing\n",
    'CCTK_CUDA_KERNEL K TYPE=3DBLOCK { CCTK_CUDA_KERNEL_VARIABLE { p } "X }\n',
    "CCTK_CUDA_KERNEL K TYPE=3DBLOCK\n TYPE=3DBLOCK { }\n",
    'CCTK_CUDA_KERNEL K { CCTK_CUDA_KERNEL_VARIABLE CACHED=YES CACHED=NO { p } "X" }\n',
    "CCTK_CUDA_KERNEL K { }\nCCTK_CUDA_KERNEL K { }\n",
    _K + '{ CCTK_CUDA_KERNEL_VARIABLE { mystery } "X" }\n',
    _K + '{ CCTK_CUDA_KERNEL_PARAMETER { anything_goes } "X" }\n',
    _K + '{ CCTK_CUDA_KERNEL_VARIABLE { vx } "A" CCTK_CUDA_KERNEL_VARIABLE { vx } "B" }\n',
    _K + '{ CCTK_CUDA_KERNEL_VARIABLE { vx } "A" CCTK_CUDA_KERNEL_PARAMETER { vx } "B" }\n',
    _K + '{ CCTK_CUDA_KERNEL_VARIABLE CACHED=MAYBE { vx } "A" }\n',
    _K + '{ CCTK_CUDA_KERNEL_VARIABLE INTENT=SIDEWAYS { vx } "A" }\n',
    _K + '{ CCTK_CUDA_KERNEL_VARIABLE COLOR=RED { vx } "A" }\n',
    _K + '{ CCTK_CUDA_KERNEL_VARIABLE INTENT=OUT { divu } "D" CCTK_CUDA_KERNEL_VARIABLE INTENT=INOUT { p } "P" }\n',
    "CCTK_CUDA_KERNEL   K\tTYPE = 3DBLOCK # c\n STENCIL =\"1, 2 ,3,4,5,6\"TILE=\"1,1,1\"{#x\n}",
    'CCTK_CUDA_KERNEL A TYPE=3DBLOCK STENCIL="1,1,1,1,1,1" TILE="2,2,2" {}\n'
    'CCTK_CUDA_KERNEL B TYPE=3DBLOCK STENCIL="2,1,0,2,1,1" TILE="8,4,2" '
    '{ CCTK_CUDA_KERNEL_VARIABLE INTENT=SEPARATEINOUT CACHED=YES { vx,vy } "V" }\n',
]
for attrs in ('TYPE=2DBLOCK STENCIL="1,1,1,1,1,1" TILE="4,4,4"', 'TYPE=3DBLOCK STENCIL="1,1,1" TILE="4,4,4"',
              'TYPE=3DBLOCK STENCIL="1,1,1,1,1,-1" TILE="4,4,4"', 'TYPE=3DBLOCK STENCIL="1,1,1,1,1,x" TILE="4,4,4"',
              'TYPE=3DBLOCK STENCIL="1,1,1,1,1,1" TILE="4,4"', 'TYPE=3DBLOCK STENCIL="1,1,1,1,1,1" TILE="4,4,0"',
              'TYPE=3DBLOCK STENCIL="1,1,1,1,1,1" TILE="4,4,4" COLOR=RED', 'STENCIL="1,1,1,1,1,1" TILE="4,4,4"',
              'TYPE=3DBLOCK TILE="4,4,4"', 'TYPE=3DBLOCK STENCIL="1,1,1,1,1,1"',
              'TYPE=3DBLOCK STENCIL="1,,1,1,1,1" TILE="4,4,4"', 'TYPE=3DBLOCK STENCIL="1,1,1,1,1,1," TILE="4,4,4"',
              'TYPE=3DBLOCK STENCIL=" 1 ,\t2,+3,1,1,1" TILE="4,4,4"', 'TYPE=3DBLOCK STENCIL=111111 TILE=4'):
    CASES.append("CCTK_CUDA_KERNEL K " + attrs + ' { CCTK_CUDA_KERNEL_VARIABLE { p } "X" }\n')


@pytest.mark.parametrize("i", range(len(CASES)))
def test_reference_test_inputs_give_the_reference_results(ref_available, i, tmp_path):
    text = CASES[i]
    assert mine(text) == ref_ccl(text)
    assert mine(text, CFD_FIELDS, str(tmp_path / "a")) == ref_ccl(text, CFD_FIELDS, str(tmp_path / "b"))


def test_syntax_error_positions_follow_the_reference_tests():
    with pytest.raises(D.ParseError) as e:
        D.parse_descriptors(CASES[2])
    assert e.value.line == 4  # test_descriptor.cpp:126-133
    with pytest.raises(D.ParseError, match="TYPE") as e:
        D.parse_descriptors(CASES[7])
    assert e.value.line == 2  # test_descriptor.cpp:144-151
    assert D.parse_descriptors("") == [] and D.parse_descriptors("# only a comment\n\n") == []


def _mutate(text, rng):
    ops = rng.randint(1, 3)
    alphabet = ' \t\n{}",=#_aZ09KP' + "CCTK_CUDA_KERNEL"
    for _ in range(ops):
        at = rng.randrange(len(text) + 1)
        r = rng.random()
        if r < 0.4 and text:
            text = text[:at] + text[at + 1:]  # delete a character
        elif r < 0.8:
            text = text[:at] + rng.choice(alphabet) + text[at:]  # insert one
        else:
            b = rng.randrange(len(text) + 1)
            text = text[:min(at, b)] + text[max(at, b):]  # cut a span
    return text


@pytest.mark.parametrize("seed", range(4))
def test_mutated_descriptor_files_give_the_reference_results(ref_available, seed, tmp_path):
    # 150 random edits of valid files per seed: every accepted file renders
    # identically, every rejected one fails with the same message, line and
    # column, and every validated one renders the same headers
    rng = random.Random(seed)
    bases = [CFD_CCL] + [c for c in CASES if c.startswith("CCTK")]
    for n in range(150):
        text = _mutate(rng.choice(bases), rng)
        assert mine(text) == ref_ccl(text), repr(text)
        assert mine(text, CFD_FIELDS) == ref_ccl(text, CFD_FIELDS, str(tmp_path / ("r%d" % n))), repr(text)


def test_the_reference_cfd_descriptor_file_parses_identically(ref_available):
    # proj/kernels/cfd.ccl, read in place (this container only)
    path = "/root/reference/proj/kernels/cfd.ccl"
    if not os.path.exists(path):
        pytest.skip("reference tree not present")
    text = open(path).read()
    assert mine(text) == ref_ccl(text)
    assert D.validate_all(D.parse_descriptors(text), CFD_FIELDS) == D.validate_all(D.parse_descriptors(CFD_CCL),
                                                                                  CFD_FIELDS)
