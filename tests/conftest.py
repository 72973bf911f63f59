"""Shared fixtures.  `-m "not gpu"` runs on CPU (oracle vs golden vectors, host logic, C-ABI
exports); `-m gpu` runs the CUDA parity tests through the C ABI on a B200."""
import json
import os
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def golden_cases():
    return sorted(p.stem for p in GOLDEN.glob("*.npz"))


def load_golden(name: str):
    """(spec, arrays, record) for one reference-generated fixture."""
    from paper_2502_15349_b200 import spec as S
    rec = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
    doc = json.loads(str(rec["doc"]))
    direct = doc.pop("rownorm_direct", None)
    spec = S.spec_from_dict(doc)
    if direct is not None:
        spec = replace(spec, rownorm=replace(spec.rownorm,
                                             direct=S.DirectRowNorm.from_source(direct)))
    arrays = {k[3:]: v for k, v in rec.items() if k.startswith("in_")}
    return spec, arrays, rec


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
