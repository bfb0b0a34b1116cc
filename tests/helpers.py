"""Shared test helpers (no GPU needed to import)."""

import hashlib
import json
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def load_npz(name):
    return np.load(os.path.join(GOLD, name))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def to_np(t) -> np.ndarray:
    if hasattr(t, "detach"):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def rel_err(a, b) -> float:
    a = to_np(a).astype(np.float64)
    b = to_np(b).astype(np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
