"""Property tests of the CPU oracle, restating the reference's own property
tests for the fused path (SURVEY §8c "Property and oracle tests"). They pin
the oracle's behaviour beyond the golden vectors: each test cites the
reference test it mirrors. CPU only, tiny config.
"""

import numpy as np
import pytest

from oracle import qcfuse_oracle as O
from tests.test_oracle_golden import load_case


@pytest.fixture(scope="module")
def tiny(golden_dir):
    z, cfg, nc = load_case(golden_dir, "tiny_case0")
    w = O.init_weights(cfg)
    chunks = [O.precompute_chunk(w, z[f"chunk{i}_tokens"], float(z["anchor_ratio"])) for i in range(nc)]
    bos = O.bos_kv(w)
    return z, cfg, w, chunks, bos, O.assemble(w, chunks, bos)


def test_rerotation_composes_with_stored_rotation():
    # test_model.py:215-225 / test_acceptance.py:82-95: R(Δ)·R(p)·x == R(p+Δ)·x to 1e-6
    rng = np.random.default_rng(3)
    x = rng.standard_normal((40, 2, 16)).astype(np.float32)
    p = np.arange(40)
    for delta in (1, 7, 513, 5121):
        a = O.rope_delta(O.rope(x, p, 10000.0), delta, 10000.0)
        b = O.rope(x, p + delta, 10000.0)
        assert np.abs(a - b).max() < 1e-5 * max(1.0, np.abs(b).max())


def test_single_chunk_fused_rows(tiny):
    # test_fusion.py:38-53: fused K = R(1)·K_c, V bit-exact, BOS row 0 (test_fusion.py:67-72)
    z, cfg, w, chunks, bos, _ = tiny
    f = O.assemble(w, chunks[:1], bos)
    assert f.offsets == [1] and f.n_ctx == chunks[0].n
    for li in range(cfg.n_layers):
        assert np.array_equal(f.keys[li][0], bos[li].keys[0])
        assert np.array_equal(f.values[li][1:], chunks[0].kv[li].values)
        assert np.abs(f.keys[li][1:] - O.rope_delta(chunks[0].kv[li].keys, 1, cfg.rope_theta)).max() < 1e-6


def test_offsets_accumulate(tiny):
    # fusion.py:241-246: offsets start at 1 and accumulate chunk lengths
    _, _, _, chunks, _, f = tiny
    assert f.offsets[0] == 1
    for a, b, c in zip(f.offsets, f.offsets[1:], chunks):
        assert b - a == c.n


def test_scores_form_a_distribution(tiny):
    # test_fusion.py:137-143: the per-key scores sum to 1
    z, cfg, w, chunks, bos, f = tiny
    pr = O.probe(w, chunks, f, z["query"], "anchors", bos, layers=cfg.critical_layer)
    c = cfg.critical_layer
    s = O.score_against_keys(pr.queries[c - 1], f.keys[c - 1][1:], cfg.d_head)
    assert s.shape == (f.n_ctx,) and (s >= 0).all()
    assert abs(float(s.sum(dtype=np.float64)) - 1.0) < 1e-5


def test_single_query_token_scores_are_one_softmax_row():
    # test_fusion.py:145-157: with one query token and one head, scores = softmax(q·K/√D)
    rng = np.random.default_rng(5)
    q = rng.standard_normal((1, 1, 8)).astype(np.float32)
    k = rng.standard_normal((30, 1, 8)).astype(np.float32)
    s = O.score_against_keys(q, k, 8)
    logits = (k[:, 0, :].astype(np.float64) @ q[0, 0].astype(np.float64)) / np.sqrt(8.0)
    e = np.exp(logits - logits.max())
    assert np.abs(s - e / e.sum()).max() < 1e-6


def test_topn_tie_rule_against_sort_oracle():
    # test_fusion.py:168-187: ties go to the lower index; result ascending and 1-based
    assert O.select_topn([0.9, 0.1, 0.5, 0.4], 0.5).tolist() == [1, 3]
    rng = np.random.default_rng(11)
    for n in (1, 7, 64, 257):
        s = rng.integers(0, 4, n).astype(np.float32) / 4  # heavy ties
        for r in (0.0, 0.1, 0.5, 1.0):
            k = int(np.ceil(r * n))
            want = sorted(sorted(range(n), key=lambda i: (-float(s[i]), i))[:k])
            assert O.select_topn(s, r).tolist() == [i + 1 for i in want]


def test_ratio_and_query_validation(tiny):
    # fusion.py:151-152, 523-530, 238: bad ratio / empty query / empty chunk list raise ValueError
    z, cfg, w, chunks, bos, f = tiny
    for r in (-0.1, 1.5):
        with pytest.raises(ValueError):
            O.select_topn([0.1, 0.2], r)
    with pytest.raises(ValueError):
        O.probe(w, chunks, f, [], "anchors", bos)
    with pytest.raises(ValueError):
        O.assemble(w, [], bos)
    with pytest.raises(ValueError):
        O.probe(w, chunks, f, z["query"], "bogus", bos)


def test_empty_selection_is_bit_identical(tiny):
    # test_fusion.py:270-278
    _, cfg, w, _, _, f = tiny
    u = O.recompute(w, f, np.zeros(0, np.int64))
    for li in range(cfg.n_layers):
        assert np.array_equal(u.keys[li], f.keys[li]) and np.array_equal(u.values[li], f.values[li])


def test_write_set_discipline(tiny):
    # test_fusion.py:280-292: only the selected rows change; the input is not mutated
    _, cfg, w, _, _, f = tiny
    before = [k.copy() for k in f.keys]
    sel = np.array([2, 5, f.n_ctx], np.int64)
    u = O.recompute(w, f, sel)
    keep = np.setdiff1d(np.arange(f.n_ctx + 1), sel)
    for li in range(cfg.n_layers):
        assert np.array_equal(f.keys[li], before[li])
        assert np.array_equal(u.keys[li][keep], f.keys[li][keep])
        assert np.array_equal(u.values[li][keep], f.values[li][keep])
        assert not np.array_equal(u.keys[li][sel], f.keys[li][sel])


def test_anchor_probe_at_full_ratio_equals_full_probe(tiny):
    # test_fusion.py:84-99: anchor_ratio 1 makes the anchor prefix the whole context
    z, cfg, w, _, bos, _ = tiny
    nc = len([k for k in z.files if k.startswith("chunk") and k.endswith("_tokens")])
    chunks = [O.precompute_chunk(w, z[f"chunk{i}_tokens"], 1.0) for i in range(nc)]
    f = O.assemble(w, chunks, bos)
    a = O.probe(w, chunks, f, z["query"], "anchors", bos)
    b = O.probe(w, chunks, f, z["query"], "full", bos)
    assert np.array_equal(a.prefix_positions, b.prefix_positions)
    for qa, qb in zip(a.queries, b.queries):
        assert np.abs(qa - qb).max() < 1e-5


def test_full_compute_recompute_equals_forward_full(tiny):
    # test_fusion.py:258-268: FullCompute's recomputed KV = forward_full over [BOS|ctx] to 1e-4
    _, cfg, w, _, _, f = tiny
    u = O.recompute(w, f, np.arange(1, f.n_ctx + 1, dtype=np.int64))
    ref = O.forward_full(w, np.concatenate([[O.BOS_ID], f.tokens]), 0)
    for li in range(cfg.n_layers):
        assert np.abs(u.keys[li] - ref.kv[li].keys).max() < 1e-4
        assert np.abs(u.values[li] - ref.kv[li].values).max() < 1e-4
