"""The reference's own unit suites run against the B200 drop-in.

oracle/_ref/conformance_b200 is proj/tests/test_*.cpp (all suites but the
CLI one), compiled unmodified, linked with libpars_b200.so (the C++ shim over
the C ABI) in place of the reference's error/features/scorer/pairs/train/
scheduler/metrics objects. conformance_ref is the same binary linked with the
reference library (harness sanity). Built by __graft_entry__.build() where
/root/reference exists; shipped prebuilt to the GPU box.
"""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden

REF_BIN = ROOT / "oracle" / "_ref" / "conformance_ref"
B200_BIN = ROOT / "oracle" / "_ref" / "conformance_b200"


def run(binary):
    # the suites write scratch files into their working directory
    import tempfile
    env = dict(os.environ, OMP_NUM_THREADS="1")
    with tempfile.TemporaryDirectory() as cwd:
        p = subprocess.run([str(binary)], capture_output=True, text=True, env=env, timeout=900,
                           cwd=cwd)
    return p.returncode, p.stdout + p.stderr


def test_reference_suites_pass_against_reference():
    if not REF_BIN.exists():
        pytest.skip("conformance_ref not built")
    rc, out = run(REF_BIN)
    assert rc == 0, out[-3000:]
    assert "test cases: 108 | passed: 108 | failed: 0" in out


@pytest.mark.gpu
def test_reference_suites_pass_against_b200_dropin():
    if not B200_BIN.exists():
        pytest.skip("conformance_b200 not built")
    rc, out = run(B200_BIN)
    assert rc == 0, out[-3000:]
    assert "test cases: 108 | passed: 108 | failed: 0" in out


@pytest.mark.gpu
def test_readme_burst_comparison_with_gpu_scored_priorities(ctx, ref):
    """README burst-500 (proj/README.md:26-36): the simulator driven by
    GPU-computed scores reproduces the reference's PARS run event for event."""
    from paper_2510_03243_b200 import Extractor, Workload
    from conftest import unhex
    g = golden("sim_burst500.json")
    w = golden("readme_model.npz")["weights"]
    wl = Workload.synthesize(500, 22)
    s = ctx.score_text(Extractor.make(), wl.text, wl.offsets, w)
    ds = ref.synthesize(500, 22)
    r = ref.simulate(ds, None, "scores", w=s)
    assert r["record"].tolist() == g["pars"]["completion"]
    assert [float(x).hex() for x in r["finish"]] == g["pars"]["finish"]
    assert float(r["mean_ms"]).hex() == g["pars"]["mean_ms"]
    assert r["iterations"] == g["pars"]["iterations"]


@pytest.mark.gpu
@pytest.mark.slow
def test_c3_poisson_100k_schedule_bit_exact(ctx, ref):
    """Config 3: 100k Poisson(5/s) requests; PARS priorities scored on the
    GPU give the identical completion order and per-request latencies as the
    CPU reference scorer (and FCFS runs alongside)."""
    from paper_2510_03243_b200 import Extractor, Workload
    z = golden("readme_model.npz")
    w = z["weights"]
    ds = ref.synthesize(100_000, 23)
    arr = ref.poisson(ds, 5.0, 24)
    wl = Workload.synthesize(100_000, 23)
    s = ctx.score_text(Extractor.make(), wl.text, wl.offsets, w)
    gpu = ref.simulate(ds, arr, "scores", w=s)
    cpu = ref.simulate(ds, arr, "pars", ex=__import__("oracle.bind", fromlist=["Extractor"]).Extractor.make(), w=w)
    assert gpu["record"].tolist() == cpu["record"].tolist()
    assert (gpu["finish"].view(np.uint64) == cpu["finish"].view(np.uint64)).all()
    assert (gpu["ptl"].view(np.uint64) == cpu["ptl"].view(np.uint64)).all()
    assert gpu["iterations"] == cpu["iterations"]


C3_B200 = ROOT / "oracle" / "_ref" / "c3_b200"


@pytest.mark.gpu
def test_c3_drop_in_simulator_bit_exact():
    """BASELINE C3 through the drop-in: the reference's own program (tools/
    c3_main.cpp, reference headers only) linked with libpars_b200 — GPU-trained
    README model, GPU-scored priorities, the incremental-queue simulator —
    reproduces the reference's FCFS and PARS runs."""
    if not C3_B200.exists():
        pytest.skip("c3_b200 not built")
    import json
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run([str(C3_B200)], capture_output=True, text=True, env=env, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["fcfs"]["completion_fnv"] == "7be6c188801b08ca"
    assert r["fcfs"]["iterations"] == 1723028
    assert float(r["fcfs"]["simulated_s"]).hex() == (19947.193749500359).hex()
    assert r["pars"]["completion_fnv"] == "322bc376a55e1141"
    assert r["pars"]["iterations"] == 1723429
    assert float(r["pars"]["mean_ms"]).hex() == (15.054321876707261).hex()
    assert float(r["pars"]["p90_ms"]).hex() == (21.624751098502799).hex()
