import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN)
                      if f.endswith(".npz") and not f.startswith(("ld_", "mca_")))
# linear discrete families other than BSC (tsc / dsc), SURVEY.md §8(f) row 2
LD_GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f.startswith("ld_"))
FAMILY_NAMES = {0: "bsc", 1: "tsc", 2: "dsc"}
# max causes (mca / mmca), SURVEY.md §8(f) row 3
MCA_GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f.startswith("mca_"))
MCA_MODES = {0: "mca", 1: "mmca"}


def golden_prior(g, pi_key="pi0", probs_key="probs0"):
    from oracle.oracle import Prior

    fam = FAMILY_NAMES[int(g["family"])]
    if fam == "dsc":
        return Prior(fam, 0.0, g["alpha"], g[probs_key])
    return Prior(fam, float(g[pi_key]))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O

    if not O.Oracle.available("port"):
        O.build()
    return O.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O

    if not O.Oracle.available("ref"):
        pytest.skip("reference build (oracle/_ref) not available")
    return O.Oracle("ref")


@pytest.fixture(autouse=True)
def _device_guards(request):
    """With BSC_GUARD=1 in the environment (guarded device allocations,
    csrc/engine_util.hpp) every GPU test ends with a check that no kernel wrote
    outside a buffer: `BSC_GUARD=1 pytest tests -m gpu` is the whole suite as an
    out-of-bounds check (compute-sanitizer is closed on this pool)."""
    yield
    if os.environ.get("BSC_GUARD") == "1" and request.node.get_closest_marker("gpu"):
        from paper_1908_06843_b200 import _native as N

        N.call("prsp_bsc_gpu_check_guards")
