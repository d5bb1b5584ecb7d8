"""The shared seeded generator: shapes and the Criteo vocabulary rule."""
import numpy as np

import synth


def test_criteo_vocab_rule():
    """the first seed s >= 0 for which
    round(exp(default_rng(s).uniform(ln 3, ln 1e7, 26))) sums into
    [3.25e7, 3.35e7] with max <= 1e7 is 230, giving CRITEO_VOCAB (total
    32,511,754; Fig. 3 of the paper quotes 33.8M rows for the real tables)."""
    for s in range(10_000):
        v = np.round(np.exp(np.random.default_rng(s).uniform(np.log(3), np.log(1e7), 26))).astype(int)
        if 3.25e7 <= v.sum() <= 3.35e7 and v.max() <= 1e7:
            break
    assert s == synth.workloads.CRITEO_VOCAB_SEED and list(v) == synth.CRITEO_VOCAB
    assert sum(synth.CRITEO_VOCAB) == 32_511_754


def test_workload_shapes_are_deterministic():
    for name in ("tiny_a", "tiny_b", "uci", "criteo", "llm"):
        a, b = synth.make_workload(name), synth.make_workload(name)
        assert all(np.array_equal(x.weights, y.weights) for x, y in zip(a.tables, b.tables))
        assert np.array_equal(a.indices, b.indices) and np.array_equal(a.dense, b.dense)
    w = synth.make_workload("criteo_b64")
    assert w.indices.shape == (64, 26)
    assert all(0 <= i < k for row in w.indices for i, k in zip(row, synth.CRITEO_VOCAB))
    llm = synth.make_workload("llm")
    assert llm.indices.shape == (1, 128) and llm.tables[0].weights.shape == (512, 768)
