"""Seeded synthetic workload generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no digit decomposition, no
encoding, no packing, no modular arithmetic): it only draws the seeded inputs
-- parameter descriptions, embedding (sub-)tables, token indices and dense
features -- with the shapes and distributions of BASELINE.json's configs.
Both `oracle/` and `paper_2506_18150_b200/` consume what it returns.

The paper's datasets (UCI Heart Disease, Criteo Kaggle, the GPT-2 table,
PAPER.md:407, :536) and trained weights are not available; these arrays stand
in for them.
"""
from .workloads import (  # noqa: F401
    CRITEO_VOCAB,
    Config,
    Table,
    Workload,
    config_by_name,
    dense_inputs,
    make_workload,
    microbench_seed,
    subtable_rows,
    CONFIG_NAMES,
)
