"""Shared test plumbing.

* registers the ``gpu`` marker (tests needing a B200 via the C-ABI library);
* loads the golden fixtures produced by the real reference
  (tests/golden/make_golden.py) into oracle problems.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from oracle import hm_oracle as orc  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the built libhubgpu.so")
    config.addinivalue_line("markers", "slow: long-running")


_cache: dict = {}


def golden(name: str):
    if name not in _cache:
        with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
            _cache[name] = {k: z[k] for k in z.files}
    return _cache[name]


def problem_from(g: dict, prefix: str) -> orc.Problem:
    n, p, chi, alpha, delta = g[f"{prefix}_meta"]
    return orc.Problem(int(n), int(p), g[f"{prefix}_dist"], g[f"{prefix}_flow"],
                       float(chi), float(alpha), float(delta))


def params_of(g: dict, label: str) -> dict:
    return json.loads(str(g[f"{label}_params"]))


GA_LABELS = ["cab", "small", "mk84", "strict", "pn", "asym", "n1", "ap", "mid", "midstrict"]
EVAL_LABELS = ["cab", "ap", "asym", "p1", "pn", "mid"]
