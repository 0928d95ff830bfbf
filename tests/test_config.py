"""Run configuration files (paper_1201_2118_b200/config.py) against the
reference's cli::parse_run_config (config.hpp, compiled in place into
oracle/_ref/libsfref.so): parsed values and error texts on hand-written cases
and on randomly mutated files. CPU only."""
import random

import pytest

from oracle.oracle import ref_parse_config
from paper_1201_2118_b200 import ConfigError
from paper_1201_2118_b200.config import ConfigFileError, load_run_config, parse_run_config

RE100 = """# Re = 100 lid-driven cavity, quasi-2D
nx = 129
ny = 129
nz = 3

re = 100
sigma = 0.9
omega = 1.9525
tolerance = 1e-6
max_sweeps = 3000
alpha = 0
tile = 129,129,3

steady_tol = 1e-6
max_steps = 200000
output_cadence = 2000

profiles_out = profiles.csv
residuals_out = residuals.csv
fields_out = fields
"""


def render(rc):
    return ("nx=%d\nny=%d\nnz=%d\nre=%.17g\nsigma=%.17g\nomega=%.17g\ntolerance=%.17g\nmax_sweeps=%d\n"
            "alpha=%.17g\ndensity=%.17g\nlid_speed=%.17g\nsymmetry_z=%d\nsteady_tol=%.17g\nmax_steps=%d\n"
            "output_cadence=%d\nworkers=%d\nmode=%s\ntile=%d,%d,%d\nghost=%d\n"
            "profiles_out=%s\nresiduals_out=%s\nfields_out=%s\n") % (
        rc.nx, rc.ny, rc.nz, rc.re, rc.sigma, rc.omega, rc.tolerance, rc.max_sweeps, rc.alpha, rc.density,
        rc.lid_speed, 1 if rc.symmetry_z else 0, rc.steady_tol, rc.max_steps, rc.output_cadence, rc.workers,
        rc.mode, rc.tile[0], rc.tile[1], rc.tile[2], rc.ghost, rc.profiles_out, rc.residuals_out, rc.fields_out)


def mine(text):
    try:
        return 0, render(parse_run_config(text))
    except ConfigFileError as e:
        return 1, str(e)
    except ConfigError as e:
        return 2, str(e)


CASES = [
    "", RE100, "nx = 17\nny=9 # c\n\tnz=2\r\n", "nx 17\n", "= 3\n", "nx = 3\nnx = 4\n", "colour = red\n",
    "nx = 0\n", "nx = 1.5\n", "nx = abc\n", "nx = 99999999999999999999\n", "re = -1\n", "re = 1e400\n",
    "re = 0x1p4\n", "re = inf\n", "re = nan\n", "re = 1e\n", "re = .5\n", "re = 5.\n", "re = +7\n", "re = 1_0\n",
    "sigma = 1\n", "omega = 2\n", "omega = 1\n", "tolerance = 0\n", "max_sweeps = 0\n", "max_sweeps = 3000000000\n",
    "alpha = 1.0000001\n", "density = 0\n", "lid_speed = 2\n", "symmetry_z = yes\n", "symmetry_z = maybe\n",
    "steady_tol = 0\n", "max_steps = -1\n", "output_cadence = -1\n", "workers = 0\n", "mode = overlap\n",
    "mode = fast\n", "tile = 1,2\n", "tile = 1,2,3,4\n", "tile = 1, 2 ,3\n", "tile = 1,2,3,\n", "tile = 1,,3\n",
    "tile = -1,2,3\n", "ghost = 0\n", "ghost = 2\n", "profiles_out = a b.csv\n", "fields_out =\n",
    "re = 100 # trailing\n", "re = 1 0\n", "nx = 08\n", "nx = -0\n", "tile = 4294967297,1,1\n",
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_config_cases_give_the_reference_results(ref_available, i):
    assert mine(CASES[i]) == ref_parse_config(CASES[i])


@pytest.mark.parametrize("seed", range(3))
def test_mutated_config_files_give_the_reference_results(ref_available, seed):
    rng = random.Random(seed)
    alphabet = " \t=#,.-+e0123456789xpna\n"
    for _ in range(300):
        text = rng.choice(CASES[1:])
        for _ in range(rng.randint(1, 3)):
            at = rng.randrange(len(text) + 1)
            if rng.random() < 0.5 and text:
                text = text[:at] + text[at + 1:]
            else:
                text = text[:at] + rng.choice(alphabet) + text[at:]
        assert mine(text) == ref_parse_config(text), repr(text)


def test_load_run_config_prefixes_the_path(tmp_path):
    p = tmp_path / "bad.cfg"
    p.write_text("nx = 1\nwhat = 2\n")
    with pytest.raises(ConfigFileError, match=r"bad.cfg: line 2: unknown key 'what'"):
        load_run_config(str(p))
    with pytest.raises(ConfigFileError, match="cannot open config file"):
        load_run_config(str(tmp_path / "missing.cfg"))
    p.write_text(RE100)
    rc = load_run_config(str(p))
    assert (rc.nx, rc.ny, rc.nz, rc.omega, rc.tile, rc.fields_out) == (129, 129, 3, 1.9525, (129, 129, 3), "fields")
