"""Helpers to load the committed golden cases (tests/golden/*.npz)."""
from __future__ import annotations

import ast
from pathlib import Path

import numpy as np

from paper_1705_09339_b200.config import EngineConfig

GOLDEN = Path(__file__).resolve().parent / "golden"

CASES = sorted(p.stem[len("case_"):] for p in GOLDEN.glob("case_*.npz"))

STATE = ("mu", "var", "w", "count", "mid_order", "mode_ref", "chp_prev",
         "last_label", "hits", "streak", "last_active", "clock", "waking",
         "group_mu", "group_var")


def load_case(name: str):
    z = np.load(GOLDEN / f"case_{name}.npz", allow_pickle=True)
    rec = {k: z[k] for k in z.files}
    overrides = {k: ast.literal_eval(v) for k, v in
                 zip(rec["cfg_keys"].tolist(), rec["cfg_vals"].tolist())}
    return rec, overrides


def config_for(overrides, **extra) -> EngineConfig:
    return EngineConfig(**{**overrides, **extra}).validate()
