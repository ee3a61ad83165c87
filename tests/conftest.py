import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def fixtures():
    from paper_2502_00778_b200 import Mesh
    with open(os.path.join(GOLDEN, "fixtures.json")) as f:
        raw = json.load(f)
    out = {}
    for name, d in raw.items():
        m = d["mesh"]
        d["mesh_obj"] = Mesh(m["dim"], m["coords"], m["elements"], m["boundary"])
        out[name] = d
    return out


@pytest.fixture(scope="session")
def golden_configs():
    from paper_2502_00778_b200 import Mesh
    z = np.load(os.path.join(GOLDEN, "configs.npz"))
    out = {}
    for name in ("C1", "C2", "C3", "C4", "C5"):
        m = Mesh(int(z[f"{name}_dim"][0]), z[f"{name}_coords"], z[f"{name}_elements"],
                 z[f"{name}_boundary"])
        out[name] = {"mesh": m, **{k[len(name) + 1:]: z[k] for k in z.files
                                   if k.startswith(name + "_")}}
    return out


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def engine():
    from paper_2502_00778_b200 import Engine
    eng = Engine()
    yield eng
    eng.close()
