import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


PIPELINE_CASES = sorted(
    os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "*.npz"))
    if os.path.basename(f).startswith(("d0_", "d1_", "d2_", "d3_", "auto_"))
    and not os.path.basename(f).startswith(("d0_kernel", "auto_params")))


def load_case(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    prm = {k[4:]: (z[k].item() if z[k].ndim == 0 else z[k]) for k in z.files if k.startswith("prm_")}
    prm["window"] = str(prm["window"])
    out = {k: z[k] for k in z.files if not k.startswith("prm_")}
    out["L"] = float(out["L"])
    out["D"] = int(out["D"])
    out["use_kernel"] = int(out["use_kernel"])
    out["prm"] = prm
    return out


@pytest.fixture(params=PIPELINE_CASES)
def golden_case(request):
    return request.param, load_case(request.param)
