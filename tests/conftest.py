import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

from paper_2003_02450_b200.graphs import Csr  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_csr(z, prefix):
    r, c = (int(x) for x in z[f"{prefix}_shape"])
    return Csr(r, c, z[f"{prefix}_indptr"], z[f"{prefix}_indices"], z[f"{prefix}_data"])


class Case:
    """One golden case produced by oracle/make_golden.py from the reference."""

    def __init__(self, name):
        meta = json.load(open(os.path.join(GOLDEN, "cases.json")))["cases"][name]
        self.name = name
        self.__dict__.update(meta)
        with np.load(os.path.join(GOLDEN, f"case_{name}.npz")) as f:
            z = {k: f[k] for k in f.files}  # eager: rank threads read it concurrently
        self.z = z
        self.h = load_csr(z, "h")
        self.ops = [load_csr(z, f"op{k}") for k in range(self.n_ops)]
        self.h_rot = load_csr(z, "hrot") if self.has_h_rot else None
        self.L = load_csr(z, "L")
        self.norms = z["norms"]
        self.rho0 = z["rho0"]

    def build_oracle(self, o):
        if self.kind == "local":
            return o.build_local(self.omega, self.h, self.ops[0], self.sources, self.sinks)
        return o.build_global(self.omega, self.h, self.ops, self.h_rot)

    def build_gpu(self, api, **kw):
        if self.kind == "local":
            return api.build_local(self.omega, self.h, self.ops[0], self.sources, self.sinks, **kw)
        return api.build_global(self.omega, self.h, self.ops, self.h_rot, **kw)


CASE_NAMES = sorted(json.load(open(os.path.join(GOLDEN, "cases.json")))["cases"])


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
