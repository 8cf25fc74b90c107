"""The reference's acceptance gate and the README burst-500 comparison, run
against the B200 drop-in.

* oracle/_ref/acceptance_{ref,b200}: proj/tests/acceptance/acceptance_main.cpp
  compiled unmodified (checks 1-12, acceptance_main.cpp:757-773) with a stub
  run_cli (oracle/stub_cli.cpp). Check 12 drives the CLI, which needs the
  absent CLI11 and is out of scope, so it must FAIL with the stub's message;
  checks 1-11 must PASS. `_ref` links the reference library, `_b200` links
  libpars_b200.so (the C++ shim over the C ABI) in place of the reference's
  features/scorer/pairs/train/scheduler/metrics/simulator objects.
* oracle/_ref/burst500_{ref,b200}: tools/burst500_main.cpp, the README's
  four-command experiment (proj/README.md:26-36) through compare_policies
  (simulator.cpp:226-283); the values are SURVEY Appendix B's.
"""
import json
import os
import re
import subprocess
import tempfile

import pytest

from conftest import ROOT

REF_DIR = ROOT / "oracle" / "_ref"

# SURVEY Appendix B, reproduced in-library from the reference
BURST500 = {
    "fcfs": {"mean_ms": 478.46399033665966, "p90_ms": 1113.5050000000272, "iterations": 6330,
             "simulated_s": 89.444600000001515},
    "oracle": {"mean_ms": 80.534870438835299, "p90_ms": 99.514409221904216, "iterations": 8855,
               "simulated_s": 94.494599999990285, "tau_b": 1.0},
    "pars": {"mean_ms": 82.853143868138957, "p90_ms": 99.721459227469552, "iterations": 8858,
             "simulated_s": 94.50059999999084, "tau_b": 0.98515882818708811},
}


def run(binary, threads="1"):
    env = dict(os.environ, OMP_NUM_THREADS=threads)
    with tempfile.TemporaryDirectory() as cwd:  # check 12 would write here
        p = subprocess.run([str(binary)], capture_output=True, text=True, env=env, timeout=1200,
                           cwd=cwd)
    return p.returncode, p.stdout, p.stderr


def parse_checks(out):
    res = {}
    for m in re.finditer(r"^\[(PASS|FAIL)\]\s+(\d+)\. ([^:]+): (.*)$", out, re.M):
        res[int(m.group(2))] = (m.group(1), m.group(3), m.group(4))
    return res


def assert_gate(binary):
    if not binary.exists():
        pytest.skip(f"{binary.name} not built")
    rc, out, err = run(binary)
    checks = parse_checks(out)
    assert sorted(checks) == list(range(1, 13)), out[-3000:] + err[-2000:]
    for k in range(1, 12):
        assert checks[k][0] == "PASS", f"check {k} ({checks[k][1]}): {checks[k][2]}"
    # check 12 is the CLI one: it fails only because run_cli is the stub
    assert checks[12][0] == "FAIL" and "CLI11 absent" in checks[12][2], checks[12]
    assert "acceptance: 11/12 passed" in out
    assert rc == 1
    return checks


def test_acceptance_gate_reference():
    """Harness sanity: the reference library passes checks 1-11."""
    assert_gate(REF_DIR / "acceptance_ref")


@pytest.mark.gpu
def test_acceptance_gate_b200_dropin():
    """The drop-in passes the reference's acceptance checks 1-11, including
    the tau brute force (:181-251), filter soundness (:257-324), SJF
    optimality (:428-483), policy equivalence (:488-525), burst HOL relief
    (:532-585) and the starvation bound (:592-652)."""
    checks = assert_gate(REF_DIR / "acceptance_b200")
    # check 10's detail line carries the README burst numbers
    assert "fcfs 478.5ms oracle 80.5ms" in checks[10][2] and "tau 0.985" in checks[10][2]


def burst(binary):
    if not binary.exists():
        pytest.skip(f"{binary.name} not built")
    rc, out, err = run(binary)
    assert rc == 0, err[-2000:]
    return json.loads(out.strip().splitlines()[-1])


def assert_burst(got):
    for pol, want in BURST500.items():
        for k, v in want.items():
            if isinstance(v, float):
                assert float(got[pol][k]).hex() == v.hex(), (pol, k, got[pol][k], v)
            else:
                assert got[pol][k] == v, (pol, k, got[pol][k], v)


def test_burst500_compare_policies_reference():
    assert_burst(burst(REF_DIR / "burst500_ref"))


@pytest.mark.gpu
def test_burst500_compare_policies_b200_dropin():
    """README burst-500 through the drop-in's compare_policies: the model is
    trained on the GPU (pars_sgd_epoch), the priorities are GPU scores, tau is
    the GPU count; every number equals the reference's bit for bit, and the
    completion order (FNV over ids + finish times) equals the reference run's."""
    got = burst(REF_DIR / "burst500_b200")
    assert_burst(got)
    ref_bin = REF_DIR / "burst500_ref"
    if ref_bin.exists():
        want = burst(ref_bin)
        for pol in ("fcfs", "oracle", "pars"):
            assert got[pol]["completion_fnv"] == want[pol]["completion_fnv"], pol
