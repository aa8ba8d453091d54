"""The op-counting instantiation of the oracle (tests/oracle_opcount.cpp):
the unchanged oracle source compiled with a counting scalar type.  Pinned on the wave RHS,
whose count follows by hand from the stencil as the oracle writes it: per D1,
(f[-2] - 8 f[-1] + 8 f[+1] - f[+2]) / (12 h) = 3 add/sub + 3 mul + 1 div; six D1 per point
(div v and grad rho) plus 2 adds for div v = 44 flops (20 add/sub, 18 mul, 6 div).  The
committed profiles/r2_oracle_opcount.jsonl (read by bench.py) must equal a fresh run."""
import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def counts(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    exe = str(tmp_path_factory.mktemp("opc") / "opcount")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I", ROOT,
                           os.path.join(ROOT, "tests", "oracle_opcount.cpp"), "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    return {d["what"]: d for d in map(json.loads, out.splitlines())}


def test_wave_rhs_count_matches_hand_count(counts):
    d = counts["wave RHS per point"]
    assert (d["add_sub"], d["mul"], d["div"], d["flops"]) == (20, 18, 6, 44)


def test_bssn_counts_are_uniform_and_committed(counts):
    rhs, step = counts["BSSN RHS per point"], counts["BSSN RK4 step per point"]
    assert rhs["exp"] == 1 and rhs["pow"] == 4      # e^{-4 phi}; alpha^n_alpha, alpha^p_beta (x3)
    assert step["flops"] > 4 * rhs["flops"]          # four RHS evaluations plus the updates
    with open(os.path.join(ROOT, "profiles", "r2_oracle_opcount.jsonl")) as fh:
        committed = {d["what"]: d for d in map(json.loads, fh.read().splitlines())}
    assert committed == counts
