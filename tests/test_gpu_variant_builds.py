"""Exact alternative forms of the kernels, each compiled here with nvcc into a
temporary directory and run through the parity tests in a subprocess
(SL_LIB_PATH) -- forms the default build takes only rarely:

* the sweep kernel's TTFT walk (`spec_walk_bounds`, csrc/sim_fast.cuh;
  reference ttft_guard, sched_scorpio.py:196-205) decides each item from two
  bounds of its sequential prefix and runs the reference's serial loop only
  for a chunk holding an item the bounds leave undecided.  Any wider margin is
  just as exact, so a 2^-2 margin sends most rejecting chunks through the
  serial form (and the recomputation of the exact prefix from the kept items):
  the golden and grid sweep parity tests must stay green on it;
* the few-large-segments guard (csrc/plan_large.cuh) certifies its CPython
  sums (sum(1/slo), vbs; sched_scorpio.py:121, 312-315) from a double-double
  sum and falls back to the sequential folds when the certificate fails --
  essentially never; SL_CERT_FOLD=0 always takes the sequential folds, and the
  config-2 plan parity tests must stay green on it.
"""

import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = {
    "wide_walk_margin": (["-DSL_WALK_MARGIN=0.25"],
                         ["tests/test_gpu_golden.py", "tests/test_gpu_sweep_parity.py"], 60),
    "sequential_folds": (["-DSL_CERT_FOLD=0"], ["tests/test_gpu_plan_parity.py"], 100),
}


@pytest.mark.parametrize("name", list(VARIANTS))
def test_variant_build_matches_reference(name, tmp_path):
    from paper_2505_23022_b200 import _native as N

    if shutil.which("nvcc") is None:
        pytest.skip("nvcc not available")
    defines, tests, min_passed = VARIANTS[name]
    lib = str(tmp_path / f"libvar_{name}.so")
    srcs = [os.path.join(N.CSRC, f) for f in N.SOURCES if os.path.exists(os.path.join(N.CSRC, f))]
    cmd = ["nvcc", *N.NVCC_FLAGS, *defines, "-I" + N.INCLUDE, "-o", lib, *srcs]
    subprocess.run(cmd, check=True, cwd=N.CSRC, timeout=900)
    env = dict(os.environ, SL_LIB_PATH=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p",
                        "no:cacheprovider", *tests],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= min_passed, r.stdout[-2000:]
