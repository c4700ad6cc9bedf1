"""End-to-end parity of the B200 engine with the reference.

Two anchors:
 * golden fixtures produced by the reference itself (tests/golden/*.npz):
   selection must be bit-exact in f32 parity mode, first-token logits within
   1e-4 (the reference's own FullCompute tolerance, test_fusion.py:299-306);
 * the CPU oracle on the same seeded inputs (fused KV, probe Q_c, scores).
The second half restates the reference's own test_fusion.py cases against the
B200 engine (same assertions, same tolerances)."""

import math
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import qcfuse_oracle as O
from tests.gpu_util import golden_setup, load_oracle_chunks

pytestmark = pytest.mark.gpu

GOLDEN = ["small_case0", "small_case1", "small_case2", "tiny_case0", "tiny_case1", "tiny_case2",
          "tiny_case3", "tiny_case4", "tiny_case5"]


@pytest.mark.parametrize("name", GOLDEN)
def test_qcfuse_fast_path_matches_reference_golden(golden_dir, tmp_path, name):
    z, oc, ow, chunks, w, store, ids, eng = golden_setup(golden_dir, name, "f32", tmp_path)
    logits, sel = eng.fuse(z["query"].tolist(), ids, float(z["ratio"]))
    assert np.array_equal(sel, z["selection"]), f"{name}: selection differs"
    assert np.abs(logits - z["first_logits"]).max() < 1e-4
    # graph replay reproduces the eager launch bit for bit
    logits2, sel2 = eng.fuse(z["query"].tolist(), ids, float(z["ratio"]))
    assert np.array_equal(sel2, sel) and np.array_equal(logits2, logits)


@pytest.mark.parametrize("name", ["small_case0", "tiny_case0"])
def test_run_matches_reference_golden_with_decode(golden_dir, tmp_path, name):
    z, oc, ow, chunks, w, store, ids, eng = golden_setup(golden_dir, name, "f32", tmp_path)
    max_new = int(z["answer"].size) if z["answer"].size > 1 else 1
    res = eng.run("QCFuse", float(z["ratio"]), ids, z["query"].tolist(), max_new=8)
    assert np.array_equal(res.selection.indices, z["selection"])
    assert np.abs(res.first_logits - z["first_logits"]).max() < 1e-4
    if name == "small_case0":
        assert res.answer_tokens == z["answer"].tolist()
    assert res.timings_ms["ttft_device_ms"] > 0


@pytest.mark.parametrize("name", ["small_case1", "tiny_case2"])
def test_stage_by_stage_vs_oracle(golden_dir, tmp_path, name):
    z, oc, ow, chunks, w, store, ids, eng = golden_setup(golden_dir, name, "f32", tmp_path)
    fused = eng.assemble_context(ids)
    ref = O.assemble(ow, chunks)
    c = oc.critical_layer
    probe = eng.probe_query(z["query"].tolist(), fused)
    assert np.array_equal(probe.prefix_positions, z["prefix_positions"])
    assert np.abs(probe.queries[c - 1] - z["q_c"]).max() < 1e-5
    scores = eng.score_critical(probe, fused)
    assert np.abs(scores - z["scores"]).max() < 1e-6
    sel = eng.select("QCFuse", float(z["ratio"]), fused, z["query"].tolist())
    assert np.array_equal(sel.indices, z["selection"])
    upd, trace = eng.recompute_selected(fused, sel)
    ref_upd = O.recompute(ow, ref, z["selection"])
    for li in range(oc.n_layers):
        assert np.abs(upd.layer_kv[li].keys - ref_upd.keys[li]).max() < 1e-4
        assert np.abs(upd.layer_kv[li].values - ref_upd.values[li]).max() < 1e-4


def test_gpu_precompute_matches_oracle(golden_dir, tmp_path):
    import paper_2604_08585_b200 as Q
    z, oc, ow, chunks, w, store, ids, eng = golden_setup(golden_dir, "small_case0", "f32", tmp_path)
    st2 = Q.ChunkStore(tmp_path / "gpu", w.config, dtype="f32")
    for i, ch in enumerate(chunks):
        rec = st2.precompute(w, ch.tokens, float(z["anchor_ratio"]))
        assert np.array_equal(rec.anchor_indices, ch.anchors)
        assert np.abs(rec.key_norms - ch.key_norms).max() < 1e-5
        for li in range(oc.n_layers):
            assert np.abs(rec.layer_kv[li].keys - ch.kv[li].keys).max() < 1e-5
            assert np.abs(rec.layer_kv[li].values - ch.kv[li].values).max() < 1e-5
    # persisted .qcfk reopens and is idempotent by hash (store.py:331-335)
    st3 = Q.ChunkStore(tmp_path / "gpu", w.config, dtype="f32")
    assert set(st3.chunk_ids()) == set(st2.chunk_ids())
    st3.precompute(w, chunks[0].tokens, float(z["anchor_ratio"]))
    assert st3.manifest.cache_hits == 1


@pytest.mark.parametrize("name", ["tiny_case0", "tiny_case3"])
def test_bf16_speed_mode_tolerance(golden_dir, tmp_path, name):
    """bf16 mode vs the reference: reported overlap + logit error bound."""
    z, oc, ow, chunks, w, store, ids, eng = golden_setup(golden_dir, name, "bf16", tmp_path)
    logits, sel = eng.fuse(z["query"].tolist(), ids, float(z["ratio"]))
    overlap = len(set(sel.tolist()) & set(z["selection"].tolist())) / len(sel)
    err = np.abs(logits - z["first_logits"]).max() / np.abs(z["first_logits"]).max()
    print(f"{name}: bf16 overlap {overlap:.3f} rel logit err {err:.3e}")
    assert overlap >= 0.85
    assert err < 5e-2


def test_fullcompute_equals_full_prefill(golden_dir, tmp_path):
    z, oc, ow, chunks, w, store, ids, eng = golden_setup(golden_dir, "small_case1", "f32", tmp_path)
    plan, b = eng.prefill("FullCompute", 1.0, ids, z["query"].tolist(), use_graph=False)
    assert np.abs(b.logits[0].cpu().numpy() - z["full_logits"]).max() < 1e-4
    logits, sel = eng.fuse(z["query"].tolist(), ids, 1.0)
    assert np.abs(logits - z["full_logits"]).max() < 1e-4


# ---------------------------------------------------------------------------
# The reference's own test_fusion.py cases, against the B200 engine
# ---------------------------------------------------------------------------

@pytest.fixture()
def engine(tmp_path):
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234)
    w = Q.init_weights(cfg, dtype="f32")
    store = Q.ChunkStore(tmp_path / "store", cfg, dtype="f32")
    return Q.FusionEngine(w, store)


@pytest.fixture()
def rng():
    return np.random.default_rng(20240811)


def seed_chunks(engine, rng, sizes=(20, 24), anchor_ratio=0.25):
    return [engine.store.precompute(engine.weights, [int(x) for x in rng.integers(0, 256, n)],
                                    anchor_ratio, "t").chunk_id for n in sizes]


class TestAssemble:
    def test_single_chunk_keys_rerotated_by_one(self, engine, rng):
        cids = seed_chunks(engine, rng, sizes=(12,))
        fused = engine.assemble_context(cids)
        rec = engine.store.get_record(cids[0])
        for li in range(engine.config.n_layers):
            expect = O.rope_delta(rec.layer_kv[li].keys, 1, engine.config.rope_theta)
            assert np.abs(fused.layer_kv[li].keys[1:] - expect).max() < 1e-6

    def test_values_copied_bit_exact(self, engine, rng):
        cids = seed_chunks(engine, rng, sizes=(10, 14))
        fused = engine.assemble_context(cids)
        r0, r1 = (engine.store.get_record(c) for c in cids)
        for li in range(engine.config.n_layers):
            stored = np.concatenate([r0.layer_kv[li].values, r1.layer_kv[li].values])
            assert np.array_equal(fused.layer_kv[li].values[1:], stored)

    def test_permuting_chunks_permutes_blocks(self, engine, rng):
        cids = seed_chunks(engine, rng, sizes=(8, 9))
        ab = engine.assemble_context(cids)
        ba = engine.assemble_context(cids[::-1])
        assert ab.offsets == [1, 9] and ba.offsets == [1, 10]
        n0 = engine.store.get_record(cids[0]).n_tokens
        assert np.array_equal(ab.token_ids[:n0], ba.token_ids[-n0:])
        assert np.array_equal(ab.layer_kv[0].values[1:1 + n0], ba.layer_kv[0].values[1 + ba.n_ctx - n0:])

    def test_empty_and_unknown_rejected(self, engine):
        with pytest.raises(ValueError):
            engine.assemble_context([])
        with pytest.raises(KeyError):
            engine.assemble_context(["ab" * 32])


class TestProbe:
    def test_full_ratio_anchor_probe_equals_full_probe(self, engine, rng):
        cids = seed_chunks(engine, rng, sizes=(16, 18), anchor_ratio=1.0)
        fused = engine.assemble_context(cids)
        q = [int(x) for x in rng.integers(0, 256, 6)]
        import paper_2604_08585_b200 as Q
        a = engine.probe_query(q, fused, Q.PROBE_ANCHORS)
        f = engine.probe_query(q, fused, Q.PROBE_FULL)
        assert np.array_equal(a.prefix_positions, f.prefix_positions)
        for x, y in zip(a.queries, f.queries):
            assert np.abs(x - y).max() < 1e-5
        assert np.abs(engine.score_critical(a, fused) - engine.score_critical(f, fused)).max() < 1e-5

    def test_probe_none_is_context_free(self, engine, rng):
        import paper_2604_08585_b200 as Q
        fused = engine.assemble_context(seed_chunks(engine, rng))
        probe = engine.probe_query([65, 66, 67, 68], fused, Q.PROBE_NONE)
        assert probe.prefix_positions.tolist() == [0]
        assert probe.critical_attention.shape[-1] == 1

    def test_anchor_positions_preserved(self, engine, rng):
        cids = seed_chunks(engine, rng, sizes=(10, 10), anchor_ratio=0.3)
        fused = engine.assemble_context(cids)
        probe = engine.probe_query([9], fused)
        r0, r1 = (engine.store.get_record(c) for c in cids)
        expect = np.concatenate([[0], 1 + r0.anchor_indices, 11 + r1.anchor_indices])
        assert probe.prefix_positions.tolist() == expect.tolist()

    def test_probe_deterministic(self, engine, rng):
        """test_fusion.py:110-117."""
        import paper_2604_08585_b200 as Q
        fused = engine.assemble_context(seed_chunks(engine, rng))
        p1 = engine.probe_query([1, 2, 3], fused, Q.PROBE_ANCHORS)
        p2 = engine.probe_query([1, 2, 3], fused, Q.PROBE_ANCHORS)
        for a, b in zip(p1.queries, p2.queries):
            assert np.array_equal(a, b)

    def test_empty_query_rejected(self, engine, rng):
        fused = engine.assemble_context(seed_chunks(engine, rng))
        with pytest.raises(ValueError):
            engine.probe_query([], fused)


class TestScoring:
    def test_single_query_token_is_one_softmax_row(self, engine, rng):
        """test_fusion.py:145-157: one query token -> the head-mean of one softmax row."""
        import paper_2604_08585_b200 as Q
        fused = engine.assemble_context(seed_chunks(engine, rng))
        probe = engine.probe_query([42], fused, Q.PROBE_FULL)
        scores = engine.score_critical(probe, fused)
        li = engine.config.critical_layer - 1
        q = probe.queries[li][0]
        keys = fused.layer_kv[li].keys[1:]
        logits = np.einsum("hd,nhd->hn", q, keys) / np.sqrt(engine.config.d_head)
        e = np.exp(logits - logits.max(axis=1, keepdims=True))
        rows = e / e.sum(axis=1, keepdims=True)
        assert np.abs(scores - rows.mean(axis=0)).max() < 1e-5

    def test_scores_sum_to_one(self, engine, rng):
        fused = engine.assemble_context(seed_chunks(engine, rng))
        scores = engine.score_critical(engine.probe_query([4, 5, 6], fused), fused)
        assert scores.shape == (fused.n_ctx,)
        assert abs(float(scores.sum()) - 1.0) < 1e-5

    def test_oracle_importance_sums_at_most_one(self, engine, rng):
        fused = engine.assemble_context(seed_chunks(engine, rng))
        s = engine.oracle_importance(fused.token_ids, [7, 8, 9])
        assert float(s.sum()) <= 1.0 + 1e-5
        assert np.array_equal(s, engine.oracle_importance(fused.token_ids, [7, 8, 9]))


class TestSelectTopN:
    def test_example(self):
        import paper_2604_08585_b200 as Q
        assert Q.select_topn(np.array([0.9, 0.1, 0.5, 0.4]), 0.5).indices.tolist() == [1, 3]

    def test_ratio_edges(self):
        import paper_2604_08585_b200 as Q
        assert Q.select_topn(np.zeros(7), 1.0).indices.tolist() == list(range(1, 8))
        assert Q.select_topn(np.ones(5), 0.0).indices.size == 0
        with pytest.raises(ValueError):
            Q.select_topn(np.ones(3), 1.5)

    def test_tie_rule_against_sort_oracle(self, rng):
        import paper_2604_08585_b200 as Q
        for _ in range(50):
            n = int(rng.integers(1, 40))
            scores = rng.choice([0.0, 0.25, 0.5, 1.0], size=n)
            ratio = float(rng.uniform(0, 1))
            got = Q.select_topn(scores, ratio).indices
            count = int(np.ceil(ratio * n))
            oracle = sorted(sorted(range(n), key=lambda i: (-scores[i], i))[:count])
            assert got.tolist() == [i + 1 for i in oracle]


class TestSparseAttention:
    @staticmethod
    def _dense_reference(q, keys, values, visible):
        """Independent dense float64 oracle (test_fusion.py:195-204)."""
        d = q.shape[-1]
        scores = np.einsum("mhd,nhd->hmn", q.astype(np.float64), keys.astype(np.float64)) / np.sqrt(d)
        scores = np.where(visible[None], scores, -np.inf)
        e = np.exp(scores - scores.max(axis=-1, keepdims=True))
        w = e / e.sum(axis=-1, keepdims=True)
        return np.einsum("hmn,nhd->mhd", w, values.astype(np.float64))

    def test_matches_dense_on_random_masks(self, rng):
        """test_fusion.py:206-217: arbitrary masks (qcf_attention_masked)."""
        import paper_2604_08585_b200 as Q
        for _ in range(100):
            m, n, h, d = int(rng.integers(1, 6)), int(rng.integers(2, 12)), 2, 8
            q = rng.normal(size=(m, h, d)).astype(np.float32)
            k = rng.normal(size=(n, h, d)).astype(np.float32)
            v = rng.normal(size=(n, h, d)).astype(np.float32)
            visible = rng.random((m, n)) < 0.6
            visible[:, 0] = True
            got = Q.sparse_attention(q, np.arange(m), k, v, visible)
            assert np.abs(got - self._dense_reference(q, k, v, visible)).max() < 1e-5

    def test_random_masks_wide_and_long(self, rng):
        """Masks over more than one 32-key word and one 32-key tile, d 64/128, GQA."""
        import paper_2604_08585_b200 as Q
        for m, n, h, d in ((7, 100, 4, 64), (40, 257, 2, 128), (3, 33, 1, 16)):
            q = rng.normal(size=(m, h, d)).astype(np.float32)
            k = rng.normal(size=(n, h, d)).astype(np.float32)
            v = rng.normal(size=(n, h, d)).astype(np.float32)
            visible = rng.random((m, n)) < 0.3
            visible[np.arange(m), rng.integers(0, n, m)] = True
            got = Q.sparse_attention(q, np.arange(m), k, v, visible)
            assert np.abs(got - self._dense_reference(q, k, v, visible)).max() < 1e-5

    def test_single_row_equals_dense_row(self, rng):
        """test_fusion.py:228-236."""
        import paper_2604_08585_b200 as Q
        n, h, d = 11, 2, 8
        q, k, v = (rng.normal(size=(n, h, d)).astype(np.float32) for _ in range(3))
        causal = np.tril(np.ones((n, n), dtype=bool))
        dense = self._dense_reference(q, k, v, causal)
        p = 6
        got = Q.sparse_attention(q[p:p + 1], np.array([p]), k, v, causal[p:p + 1])
        assert np.abs(got[0] - dense[p]).max() < 1e-5

    def test_key_permutation_equivariance(self, rng):
        """test_fusion.py:238-248."""
        import paper_2604_08585_b200 as Q
        m, n, h, d = 3, 8, 2, 8
        q = rng.normal(size=(m, h, d)).astype(np.float32)
        k = rng.normal(size=(n, h, d)).astype(np.float32)
        v = rng.normal(size=(n, h, d)).astype(np.float32)
        visible = rng.random((m, n)) < 0.7
        visible[:, 0] = True
        perm = rng.permutation(n)
        a = Q.sparse_attention(q, np.arange(m), k, v, visible)
        b = Q.sparse_attention(q, np.arange(m), k[perm], v[perm], visible[:, perm])
        assert np.abs(a - b).max() < 1e-6

    def test_full_mask_equals_dense_causal(self, rng):
        import paper_2604_08585_b200 as Q
        n, h, d = 9, 2, 8
        q, k, v = (rng.normal(size=(n, h, d)).astype(np.float32) for _ in range(3))
        causal = np.tril(np.ones((n, n), dtype=bool))
        got = Q.sparse_attention(q, np.arange(n), k, v, causal)
        ref, _ = O.attention(q, k, v, causal)
        assert np.abs(got - ref).max() < 1e-5

    def test_empty_visible_rejected(self, rng):
        import paper_2604_08585_b200 as Q
        q = rng.normal(size=(1, 2, 8)).astype(np.float32)
        k = rng.normal(size=(4, 2, 8)).astype(np.float32)
        with pytest.raises(ValueError):
            Q.sparse_attention(q, np.array([0]), k, k, np.zeros((1, 4), dtype=bool))


class TestRecompute:
    def test_full_selection_matches_forward_full(self, engine, rng):
        cids = seed_chunks(engine, rng, sizes=(16, 20))
        fused = engine.assemble_context(cids)
        upd, _ = engine.recompute_selected(fused, engine.select("FullCompute", 1.0, fused, [1]))
        ow = O.init_weights(O.Config(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234))
        full = O.forward_full(ow, np.concatenate([[256], fused.token_ids]), 0)
        for li in range(engine.config.n_layers):
            assert np.abs(upd.layer_kv[li].keys - full.kv[li].keys).max() < 1e-4
            assert np.abs(upd.layer_kv[li].values - full.kv[li].values).max() < 1e-4

    def test_empty_selection_bit_identical(self, engine, rng):
        fused = engine.assemble_context(seed_chunks(engine, rng))
        upd, trace = engine.recompute_selected(fused, engine.select("FullReuse", 0.0, fused, [1]))
        for li in range(engine.config.n_layers):
            assert np.array_equal(upd.layer_kv[li].keys, fused.layer_kv[li].keys)
            assert np.array_equal(upd.layer_kv[li].values, fused.layer_kv[li].values)
        assert all(c == 0.0 for c in trace.compute_seconds)

    def test_write_set_discipline(self, engine, rng):
        fused = engine.assemble_context(seed_chunks(engine, rng, sizes=(18, 22)))
        sel = engine.select("Random", 0.3, fused, [1])
        upd, _ = engine.recompute_selected(fused, sel)
        outside = np.setdiff1d(np.arange(0, fused.n_ctx + 1), sel.indices)
        for li in range(engine.config.n_layers):
            assert np.array_equal(upd.layer_kv[li].keys[outside], fused.layer_kv[li].keys[outside])
            assert np.array_equal(upd.layer_kv[li].values[outside], fused.layer_kv[li].values[outside])
            assert not np.array_equal(upd.layer_kv[li].keys[sel.indices], fused.layer_kv[li].keys[sel.indices])


class TestRun:
    def test_fullcompute_equals_pure_forward(self, engine, rng):
        res = engine.run("FullCompute", 1.0, seed_chunks(engine, rng), "what?", compare_oracle=True)
        assert res.comparison.logit_div_max < 1e-4
        assert res.comparison.token_match == 1.0

    def test_qcfuse_ratio_one_equals_fullcompute(self, engine, rng):
        cids = seed_chunks(engine, rng)
        qc = engine.run("QCFuse", 1.0, cids, "same answer")
        fc = engine.run("FullCompute", 1.0, cids, "same answer")
        assert np.abs(qc.first_logits - fc.first_logits).max() < 1e-4
        assert qc.answer_tokens == fc.answer_tokens

    def test_run_deterministic(self, engine, rng):
        cids = seed_chunks(engine, rng)
        r1 = engine.run("QCFuse", 0.3, cids, "again", compare_oracle=True)
        r2 = engine.run("QCFuse", 0.3, cids, "again", compare_oracle=True)
        assert r1.answer_tokens == r2.answer_tokens
        assert np.array_equal(r1.selection.indices, r2.selection.indices)
        assert r1.ttft_sim == r2.ttft_sim

    def test_selection_excludes_bos(self, engine, rng):
        cids = seed_chunks(engine, rng)
        n_ctx = engine.assemble_context(cids).n_ctx
        for pol in ("QCFuse", "Random", "EPIC", "QCLast", "QCAll"):
            res = engine.run(pol, 0.4, cids, "bounds")
            assert res.selection.indices.min() >= 1 and res.selection.indices.max() <= n_ctx

    def test_event_timestamps_match_schedule(self, engine, rng):
        res = engine.run("QCFuse", 0.2, seed_chunks(engine, rng), "events")
        comp = [e for e in res.trace.events if e["kind"] == "compute"]
        assert len(comp) == engine.config.n_layers
        assert [e["end"] for e in comp] == res.schedule.compute_end

    def test_invalid_inputs(self, engine, rng):
        cids = seed_chunks(engine, rng)
        for args in (("Nope", 0.2, cids, "x"), ("QCFuse", 1.2, cids, "x"), ("QCFuse", 0.2, cids, "")):
            with pytest.raises(ValueError):
                engine.run(*args)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_batched_prefill_equals_single_requests(tmp_path, dtype):
    """A homogeneous batch of requests (config 3) gives every request the
    selection and first-token logits it gets alone (f32: bit-exact)."""
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=4, d_model=512, d_head=128, d_ff=1024, seed=99)
    w = Q.init_weights(cfg, dtype=dtype)
    store = Q.ChunkStore(tmp_path / "s", cfg, dtype=dtype, persist=False)
    eng = Q.FusionEngine(w, store)
    pool = [store.precompute(w, np.random.default_rng(i).integers(0, 256, 96), 0.05).chunk_id for i in range(6)]
    rng = np.random.default_rng(3)
    reqs = [[pool[j] for j in rng.permutation(6)[:3]] for _ in range(4)]
    queries = [rng.integers(0, 256, 12).tolist() for _ in range(4)]
    plans, b = eng.prefill_batch("QCFuse", 0.2, reqs, queries, use_graph=True)
    n_sel = plans[0].n_sel
    for r in range(4):
        logits, sel = eng.fuse(queries[r], reqs[r], 0.2)
        bsel = b.rc_pos[r * b.Mr:r * b.Mr + n_sel].cpu().numpy()
        blog = b.logits[r].cpu().numpy()
        if dtype == "f32":
            assert np.array_equal(bsel, sel) and np.array_equal(blog, logits)
        else:
            assert len(set(bsel.tolist()) & set(sel.tolist())) >= 0.9 * n_sel
            assert np.abs(blog - logits).max() < 5e-2 * np.abs(logits).max()


@pytest.mark.parametrize("knob", [4, 8])
def test_batched_prefill_attention_kernels(tmp_path, knob):
    """The batch's attention kernels inside the engine: a bf16 batch run with the
    two-CTAs-per-SM kernel (knob 4, the auto choice for the benchmarked batch) or
    the two-softmax-group kernel (knob 8) tracks each request's single-request run
    (single-tile kernel) within the bf16 tolerance of the batched test above."""
    import paper_2604_08585_b200 as Q
    from paper_2604_08585_b200 import _lib
    cfg = Q.ModelConfig(n_layers=4, n_heads=4, d_model=512, d_head=128, d_ff=1024, seed=97)
    w = Q.init_weights(cfg, dtype="bf16")
    store = Q.ChunkStore(tmp_path / "s", cfg, dtype="bf16", persist=False)
    eng = Q.FusionEngine(w, store)
    pool = [store.precompute(w, np.random.default_rng(i).integers(0, 256, 256), 0.05).chunk_id for i in range(6)]
    rng = np.random.default_rng(7)
    reqs = [[pool[j] for j in rng.permutation(6)[:4]] for _ in range(4)]
    queries = [rng.integers(0, 256, 16).tolist() for _ in range(4)]
    singles = [eng.fuse(queries[r], reqs[r], 0.2) for r in range(4)]
    _lib.call("qcf_set_attention_kernel", knob)
    try:
        plans, b = eng.prefill_batch("QCFuse", 0.2, reqs, queries, use_graph=False)
        torch.cuda.synchronize()
    finally:
        _lib.call("qcf_set_attention_kernel", 0)
    n_sel = plans[0].n_sel
    for r, (logits, sel) in enumerate(singles):
        bsel = b.rc_pos[r * b.Mr:r * b.Mr + n_sel].cpu().numpy()
        blog = b.logits[r].cpu().numpy()
        assert len(set(bsel.tolist()) & set(sel.tolist())) >= 0.9 * n_sel, r
        assert np.abs(blog - logits).max() < 5e-2 * np.abs(logits).max(), r


# ---------------------------------------------------------------- GQA extension (BASELINE configs[3] shape family)
def _gqa_case(tmp_path, dtype, H, Hkv, D, d_ff, lens, q, ratio, seed=5):
    import paper_2604_08585_b200 as Q
    from tests.gpu_util import device_weights
    oc = O.Config(n_layers=4, n_heads=H, n_kv_heads=Hkv, d_model=H * D, d_head=D, d_ff=d_ff, seed=seed)
    ow = O.init_weights(oc)
    rng = np.random.default_rng(seed)
    chunks = [O.precompute_chunk(ow, rng.integers(0, 256, n), 0.1) for n in lens]
    query = rng.integers(0, 256, q).tolist()
    ref = O.run(ow, chunks, query, ratio)
    w = device_weights(ow, dtype)
    store = Q.ChunkStore(tmp_path / "s", w.config, dtype=dtype, persist=False)
    ids = load_oracle_chunks(store, chunks)
    eng = Q.FusionEngine(w, store)
    logits, sel = eng.fuse(query, ids, ratio)
    return ref, logits, sel, oc, ow


@pytest.mark.parametrize("H,Hkv", [(4, 2), (4, 1), (8, 2)])
def test_gqa_f32_matches_oracle(tmp_path, H, Hkv):
    """GQA in the f32 parity mode: selection bit-exact and first-token logits
    within 1e-4 of the oracle restatement (which reduces to the reference at
    Hkv == H and repeats kv heads otherwise)."""
    ref, logits, sel, _, _ = _gqa_case(tmp_path, "f32", H, Hkv, 16, 128, [40, 33, 51], 8, 0.25)
    assert np.array_equal(sel, ref.selection)
    assert np.abs(logits - ref.first_logits).max() < 1e-4


def test_gqa_bf16_tensor_core_path(tmp_path):
    """GQA-4 at D=128 runs the tcgen05 GEMM / attention / scoring kernels;
    bf16 speed-mode bounds vs the f32 oracle (overlap >= 0.85, rel logit err < 5e-2)."""
    ref, logits, sel, _, _ = _gqa_case(tmp_path, "bf16", 8, 2, 128, 2048, [160, 128, 192], 32, 0.15)
    overlap = len(set(sel.tolist()) & set(ref.selection.tolist())) / len(sel)
    err = np.abs(logits - ref.first_logits).max() / np.abs(ref.first_logits).max()
    print(f"GQA bf16 overlap {overlap:.3f} rel logit err {err:.3e}")
    assert overlap >= 0.85 and err < 5e-2


def test_gqa_init_bit_exact(tmp_path):
    """On-device splitmix64 init with GQA wk/wv shapes equals the oracle's draws."""
    import paper_2604_08585_b200 as Q
    from paper_2604_08585_b200.model import untile64
    cfg = Q.ModelConfig(n_layers=4, n_heads=8, n_kv_heads=2, d_model=512, d_head=64, d_ff=256, seed=77)
    w = Q.init_weights(cfg, dtype="f32")
    ow = O.init_weights(O.Config(n_layers=4, n_heads=8, n_kv_heads=2, d_model=512, d_head=64, d_ff=256, seed=77))
    for li in (0, 3):
        wqkv = w.layers[li].wqkv.cpu().numpy()
        ref = np.concatenate([ow.layers[li].wq, ow.layers[li].wk, ow.layers[li].wv], axis=1).T
        assert np.array_equal(wqkv, ref)
        assert np.array_equal(w.layers[li].w2.cpu().numpy(), ow.layers[li].w2.T)


# ---------------------------------------------------------------- comparison policies
@pytest.mark.parametrize("name", ["small", "small2", "tiny"])
def test_baseline_policies_match_reference(tmp_path, name):
    """QCLast / QCAll select exactly the reference's index sets in the f32
    parity mode; the layer-1 pass reproduces the reference's received attention
    (1e-6) and its KV deviations to noise level. In the reference model layer-1
    K/V do not depend on context (only on the token and a rotation), so an
    untouched cache has deviations of pure rounding noise (~1e-7) and the
    CacheBlend / KVShare ranking of such a cache is decided by BLAS rounding
    order -- not reproducible across implementations; the perturbed-cache test
    below pins those two policies where the deviation carries signal."""
    import json
    from pathlib import Path
    import paper_2604_08585_b200 as Q
    from tests.gpu_util import device_weights
    z = np.load(Path(__file__).parent / "golden" / "baselines.npz")
    d = json.loads(str(z[f"{name}_cfg"]))
    oc = O.Config(**{k: d[k] for k in ("n_layers", "n_heads", "d_model", "d_head", "d_ff", "rope_theta", "ln_eps",
                                       "seed", "critical_layer")})
    ow = O.init_weights(oc)
    chunks = [O.precompute_chunk(ow, z[f"{name}_chunk{i}_tokens"], 0.1) for i in range(int(z[f"{name}_n_chunks"]))]
    w = device_weights(ow, "f32")
    store = Q.ChunkStore(tmp_path / "s", w.config, dtype="f32", persist=False)
    ids = load_oracle_chunks(store, chunks)
    eng = Q.FusionEngine(w, store)
    fused = eng.assemble_context(ids)
    k, v, received = eng._layer1_recompute_pass(fused, want_attention=True)
    dev = eng._kv_deviation(fused, k, v).cpu().numpy()
    assert np.abs(dev - z[f"{name}_deviation"]).max() < 1e-5
    assert np.abs(received.cpu().numpy() - z[f"{name}_received"]).max() < 1e-6
    r = float(z[f"{name}_ratio"])
    q = z[f"{name}_query"].tolist()
    for pol in ("QCLast", "QCAll"):
        got = eng.select(pol, r, fused, q).indices
        assert np.array_equal(got, z[f"{name}_{pol}"]), pol
    for pol in ("CacheBlend", "KVShare"):   # well-formed selections
        got = eng.select(pol, r, fused, q).indices
        assert got.size == math.ceil(r * fused.n_ctx) and np.all(np.diff(got) > 0)
        assert got.min() >= 1 and got.max() <= fused.n_ctx


def test_cacheblend_kvshare_on_stale_cache_match_oracle(tmp_path):
    """A stale chunk cache (layer-1 K/V of 30% of the rows perturbed, as if
    computed under another context): CacheBlend / KVShare on the GPU select
    exactly the oracle's index sets (deviation and received attention carry
    the signal), through select() and through run()."""
    import paper_2604_08585_b200 as Q
    from tests.gpu_util import device_weights
    oc = O.Config(n_layers=4, n_heads=4, d_model=256, d_head=64, d_ff=1024, seed=1234)
    ow = O.init_weights(oc)
    rng = np.random.default_rng(7)
    chunks = [O.precompute_chunk(ow, rng.integers(0, 256, 96), 0.1) for _ in range(3)]
    for ch in chunks:
        rows = rng.permutation(96)[:29]
        ch.kv[0].keys[rows] += rng.normal(0, 0.5, ch.kv[0].keys[rows].shape).astype(np.float32)
        ch.kv[0].values[rows] += rng.normal(0, 0.5, ch.kv[0].values[rows].shape).astype(np.float32)
    fused_o = O.assemble(ow, chunks)
    w = device_weights(ow, "f32")
    store = Q.ChunkStore(tmp_path / "s", w.config, dtype="f32", persist=False)
    ids = load_oracle_chunks(store, chunks)
    eng = Q.FusionEngine(w, store)
    fused = eng.assemble_context(ids)
    q = rng.integers(0, 256, 8).tolist()
    for ratio in (0.1, 0.25):
        assert np.array_equal(eng.select("CacheBlend", ratio, fused, q).indices,
                              O.select_topn(O.cacheblend_scores(ow, fused_o), ratio))
        assert np.array_equal(eng.select("KVShare", ratio, fused, q).indices,
                              O.select_topn(O.kvshare_scores(ow, fused_o), ratio))
    res = eng.run("CacheBlend", 0.25, ids, q, max_new=1)
    assert np.array_equal(res.selection.indices, O.select_topn(O.cacheblend_scores(ow, fused_o), 0.25))


def test_received_attention_row_chunking(tmp_path):
    """qcf_received_attention gives the same column means whether all rows fit
    the workspace or are processed in many chunks (bf16 inputs, GQA)."""
    from paper_2604_08585_b200 import _lib as L
    torch.manual_seed(0)
    n, H, Hkv, D = 300, 8, 2, 128
    q = (torch.randn(n, H, D, device="cuda") * 0.5).bfloat16()
    k = (torch.randn(n + 1, Hkv, D, device="cuda") * 0.5).bfloat16()
    pos = torch.arange(1, n + 1, dtype=torch.int32, device="cuda")
    outs = []
    for rows_fit in (n, 7):
        ws_bytes = 8 * (n + 1) + 256 + rows_fit * 8 * (H * (n + 1) + 2 * H)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
        out = torch.empty(n + 1, device="cuda")
        L.call("qcf_received_attention", L.QCF_BF16, q.data_ptr(), k.data_ptr(), n + 1, n, H, Hkv, D,
               1.0 / math.sqrt(D), pos.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(),
               torch.cuda.current_stream().cuda_stream)
        outs.append(out.cpu().numpy())
    kk = k.float().repeat_interleave(H // Hkv, dim=1)
    s = torch.einsum("thd,nhd->htn", q.float(), kk) / math.sqrt(D)
    mask = torch.arange(n + 1, device="cuda")[None, :] <= pos[:, None]
    ref = torch.softmax(s.masked_fill(~mask[None], float("-inf")), dim=-1).mean(dim=(0, 1)).cpu().numpy()
    assert np.abs(outs[0] - ref).max() < 1e-6
    assert np.abs(outs[1] - outs[0]).max() < 1e-7


# ---------------------------------------------------------------- host-pool tier
@pytest.mark.parametrize("dtype,policy", [("f32", "QCFuse"), ("bf16", "QCFuse"), ("bf16", "FullCompute")])
def test_host_pool_pipelined_equals_hbm_pool(tmp_path, dtype, policy):
    """Chunk KV in pinned host memory, streamed layer by layer while the
    previous layer recomputes: selection and first-token logits bit-identical to
    the HBM-resident pool (same kernels, same arithmetic), single and batched."""
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=4, d_model=512, d_head=128, d_ff=1024, seed=21)
    w = Q.init_weights(cfg, dtype=dtype)
    hbm = Q.ChunkStore(tmp_path / "a", cfg, dtype=dtype, persist=False)
    host = Q.ChunkStore(tmp_path / "b", cfg, dtype=dtype, persist=False, pool="host")
    toks = [np.random.default_rng(40 + i).integers(0, 256, 96) for i in range(4)]
    ids = [hbm.precompute(w, t, 0.05).chunk_id for t in toks]
    for cid in ids:
        r = hbm.get_record(cid)
        host.add_record(r.token_ids, r.k, r.v, r.key_norms, r.anchor_indices)
    assert host.get_record(ids[0]).on_host and host.get_record(ids[0]).anchor_k.is_cuda
    e1, e2 = Q.FusionEngine(w, hbm), Q.FusionEngine(w, host)
    rng = np.random.default_rng(5)
    reqs = [[ids[j] for j in rng.permutation(4)[:3]] for _ in range(3)]   # equal chunk lengths: one batch shape
    qs = [rng.integers(0, 256, 12).tolist() for _ in range(3)]
    p1, b1 = e1.prefill_batch(policy, 0.2, reqs, qs, use_graph=False)
    l1, s1 = b1.logits.cpu().numpy().copy(), b1.rc_pos.cpu().numpy().copy()
    p2, b2 = e2.prefill_batch(policy, 0.2, reqs, qs)
    torch.cuda.synchronize()
    assert np.array_equal(b2.rc_pos.cpu().numpy(), s1)
    assert np.array_equal(b2.logits.cpu().numpy(), l1)
    lg, sel = e2.fuse(qs[0], reqs[0], 0.2)
    lg1, sel1 = e1.fuse(qs[0], reqs[0], 0.2)
    assert np.array_equal(sel, sel1) and np.array_equal(lg, lg1)


def test_llama_width_bf16_against_oracle(tmp_path):
    """Full Llama-3-8B WIDTH (d 4096, H 32, D 128, F 14336) at the reference's
    minimum depth (L 4), 2 x 512-token chunks, q 32, r .15: the bf16 speed
    path (tcgen05 GEMMs / attention / scoring) against the f32 oracle on the
    same splitmix64 weights and the same chunk KV. Bounds: Top-N overlap >= 0.9,
    relative first-token logit error < 5e-2, same top-1 token."""
    import paper_2604_08585_b200 as Q
    from tests.gpu_util import device_weights
    oc = O.Config(n_layers=4, n_heads=32, d_model=4096, d_head=128, d_ff=14336, seed=1234)
    ow = O.init_weights(oc)
    rng = np.random.default_rng(2024)
    chunks = [O.precompute_chunk(ow, rng.integers(0, 256, 512), 0.05) for _ in range(2)]
    query = rng.integers(0, 256, 32).tolist()
    ref = O.run(ow, chunks, query, 0.15)
    w = device_weights(ow, "bf16")
    store = Q.ChunkStore(tmp_path / "s", w.config, dtype="bf16", persist=False)
    ids = load_oracle_chunks(store, chunks)
    eng = Q.FusionEngine(w, store)
    logits, sel = eng.fuse(query, ids, 0.15)
    overlap = len(set(sel.tolist()) & set(ref.selection.tolist())) / len(sel)
    err = np.abs(logits - ref.first_logits).max() / np.abs(ref.first_logits).max()
    print(f"Llama width L4: overlap {overlap:.3f} rel logit err {err:.3e}")
    assert overlap >= 0.9 and err < 5e-2
    assert int(np.argmax(logits)) == int(np.argmax(ref.first_logits))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_precompute_batch_equals_precompute(tmp_path, dtype):
    """Batched chunk precompute (one layer stack over B equal-length chunks)
    produces the same records as one-at-a-time precompute: K/V bit-identical
    (bf16 chunks of <= 64 tokens precomputed ALONE take the split-K weight-
    streaming GEMM, whose fp32 sums associate differently: equal to bf16
    rounding there), same anchors, cache hits for known chunks, mixed lengths grouped."""
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=4, d_model=512, d_head=128, d_ff=1024, seed=5)
    w = Q.init_weights(cfg, dtype=dtype)
    rng = np.random.default_rng(1)
    toks = [rng.integers(0, 256, n) for n in (96, 96, 64, 96, 64)]
    s1 = Q.ChunkStore(tmp_path / "a", cfg, dtype=dtype, persist=False)
    s2 = Q.ChunkStore(tmp_path / "b", cfg, dtype=dtype, persist=False)
    r1 = [s1.precompute(w, t, 0.1) for t in toks]
    s2.precompute(w, toks[1], 0.1)                    # one already cached
    r2 = s2.precompute_batch(w, toks + [toks[0]], 0.1)
    assert s2.manifest.cache_hits == 2                # the cached chunk + the in-call duplicate
    for t, a, b in zip(toks, r1, r2):
        assert a.chunk_id == b.chunk_id
        assert np.array_equal(a.anchor_indices, b.anchor_indices)
        if dtype == "bf16" and len(t) <= 64:
            for x, y in ((a.k, b.k), (a.v, b.v)):
                assert (x.float() - y.float()).abs().max().item() <= 2 ** -6 * max(1.0, y.float().abs().max().item())
        else:
            assert torch.equal(a.k, b.k) and torch.equal(a.v, b.v)
    assert r2[-1].chunk_id == r1[0].chunk_id


def test_engine_is_reentrant_across_threads(tmp_path):
    """The reference engine may be shared by threads (fusion.py:211-216, the
    FastAPI threadpool): concurrent fuse() calls give the sequential results."""
    import threading
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=4, d_model=512, d_head=128, d_ff=1024, seed=8)
    w = Q.init_weights(cfg, dtype="bf16")
    store = Q.ChunkStore(tmp_path / "s", cfg, dtype="bf16", persist=False)
    ids = [store.precompute(w, np.random.default_rng(i).integers(0, 256, 80), 0.05).chunk_id for i in range(3)]
    eng = Q.FusionEngine(w, store)
    qs = [np.random.default_rng(100 + i).integers(0, 256, 8).tolist() for i in range(6)]
    ref = [eng.fuse(q, ids, 0.2) for q in qs]
    got = [None] * len(qs)

    def work(i):
        got[i] = eng.fuse(qs[i], ids, 0.2)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(qs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for (l1, s1), (l2, s2) in zip(ref, got):
        assert np.array_equal(s1, s2) and np.array_equal(l1, l2)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_long_context_16k_against_oracle(tmp_path, dtype):
    """16 chunks x 1024 tokens (16k context, RoPE table growth, 129 key tiles,
    16k-key Top-N and scoring) through the fast path vs the oracle. f32: the
    selection is bit-exact and logits within 1e-4; bf16: overlap >= 0.9 and
    relative logit error < 5e-2."""
    import paper_2604_08585_b200 as Q
    from tests.gpu_util import device_weights
    oc = O.Config(n_layers=4, n_heads=4, d_model=512, d_head=128, d_ff=1024, seed=31)
    ow = O.init_weights(oc)
    rng = np.random.default_rng(16)
    chunks = [O.precompute_chunk(ow, rng.integers(0, 256, 1024), 0.05) for _ in range(16)]
    query = rng.integers(0, 256, 24).tolist()
    ref = O.run(ow, chunks, query, 0.15)
    w = device_weights(ow, dtype)
    store = Q.ChunkStore(tmp_path / "s", w.config, dtype=dtype, persist=False)
    ids = load_oracle_chunks(store, chunks)
    eng = Q.FusionEngine(w, store)
    logits, sel = eng.fuse(query, ids, 0.15)
    if dtype == "f32":
        assert np.array_equal(sel, ref.selection)
        assert np.abs(logits - ref.first_logits).max() < 1e-4
    else:
        overlap = len(set(sel.tolist()) & set(ref.selection.tolist())) / len(sel)
        err = np.abs(logits - ref.first_logits).max() / np.abs(ref.first_logits).max()
        print(f"16k bf16: overlap {overlap:.3f} rel logit err {err:.3e}")
        assert overlap >= 0.9 and err < 5e-2


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_graph_decode_equals_eager_decode(golden_dir, tmp_path, dtype):
    """Greedy decode as a replayed CUDA graph with the argmax on the device
    (qcf_decode_advance, np.argmax's tie rule) gives the eager loop's tokens
    (model.py:433-465); f32 also equals the reference's golden answer."""
    z, oc, ow, chunks, w, store, ids, eng = golden_setup(golden_dir, "small_case0", dtype, tmp_path)
    outs = []
    for graph in (True, False, True):
        eng.decode_graph = graph
        res = eng.run("QCFuse", float(z["ratio"]), ids, z["query"].tolist(), max_new=12)
        outs.append(res.answer_tokens)
    eng.decode_graph = True
    assert outs[0] == outs[1] == outs[2]
    assert 1 <= len(outs[0]) <= 12
    if dtype == "f32":
        n = min(len(outs[0]), z["answer"].size)
        assert outs[0][:n] == z["answer"].tolist()[:n]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_side_stream_assembly_matches_serial(golden_dir, tmp_path, dtype):
    """The assembly on a side stream by layer ranges (joined layer by layer by the
    recompute; graph-captured fork/join) gives bit-identical logits and selections
    to the serial main-stream assembly, eager and graph replay."""
    z, oc, ow, chunks, w, store, ids, eng = golden_setup(golden_dir, "small_case0", dtype, tmp_path)
    out = []
    for pipe, graph in ((False, False), (True, False), (True, True), (False, True)):
        eng.pipeline_asm = pipe
        eng._bufs.clear()
        plan, b = eng.prefill("QCFuse", float(z["ratio"]), ids, z["query"].tolist(), use_graph=graph)
        torch.cuda.synchronize()
        out.append((b.logits[0].cpu().clone(), b.rc_pos[:plan.n_sel].cpu().clone()))
    eng.pipeline_asm = True
    for lg, sel in out[1:]:
        assert torch.equal(lg, out[0][0]) and torch.equal(sel, out[0][1])


def test_rope_growth_keeps_captured_graphs_correct(tmp_path):
    """fuse() at a 5k context (graph captured), then at 16k (the RoPE table
    grows past its initial 8192 positions and moves), then the 5k request
    again: the replayed graph must give bit-identical logits and selection."""
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=256, d_head=128, d_ff=512, seed=11)
    w = Q.init_weights(cfg, dtype="bf16")
    store = Q.ChunkStore(tmp_path, cfg, dtype="bf16", persist=False)
    rng = np.random.default_rng(3)
    pool = [store.precompute(w, rng.integers(0, 256, 512)).chunk_id for _ in range(32)]
    eng = Q.FusionEngine(w, store)
    query = rng.integers(0, 256, 16).tolist()
    small = pool[:10]
    l1, s1 = eng.fuse(query, small, 0.15)
    ptr0 = eng.ex.rope.cos.data_ptr()
    l_big, s_big = eng.fuse(query, pool, 0.15)          # 16384 context rows
    assert eng.ex.rope.n_pos > 8192 and eng.ex.rope.cos.data_ptr() != ptr0
    l2, s2 = eng.fuse(query, small, 0.15)
    assert np.array_equal(s1, s2) and np.array_equal(l1, l2)
    # a fresh engine (no captured graph) agrees with the replayed one
    eng2 = Q.FusionEngine(w, store)
    l3, s3 = eng2.fuse(query, small, 0.15)
    assert np.array_equal(s1, s3) and np.array_equal(l1, l3)


def test_shape_cache_is_bounded_lru(tmp_path):
    """At most max_shapes per-shape buffer sets stay resident; an evicted
    shape is rebuilt with identical results."""
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=256, d_head=128, d_ff=512, seed=12)
    w = Q.init_weights(cfg, dtype="bf16")
    store = Q.ChunkStore(tmp_path, cfg, dtype="bf16", persist=False)
    rng = np.random.default_rng(4)
    ids = [store.precompute(w, rng.integers(0, 256, 128)).chunk_id for _ in range(4)]
    eng = Q.FusionEngine(w, store)
    eng.max_shapes = 2
    q = rng.integers(0, 256, 8).tolist()
    first = eng.fuse(q, ids[:2], 0.2)
    eng.fuse(q, ids[:3], 0.2)
    eng.fuse(q, ids[:4], 0.2)
    assert len(eng._bufs) == 2
    again = eng.fuse(q, ids[:2], 0.2)
    assert len(eng._bufs) == 2
    assert np.array_equal(first[0], again[0]) and np.array_equal(first[1], again[1])


def test_ratio_one_oracle_equivalence_20_seeds(tmp_path):
    """test_acceptance.py:54-79 against the B200 engine (f32 parity mode):
    QCFuse at ratio 1.0 reproduces full computation -- first logits within
    1e-4 and a 100% 32-token greedy match over 20 seeded cases, under 60 s --
    and additionally matches the CPU oracle's full prefill to 1e-4."""
    import time

    import paper_2604_08585_b200 as Q
    started = time.time()
    for case in range(20):
        rng = np.random.default_rng(case)
        cfg = Q.ModelConfig(seed=3000 + case)
        w = Q.init_weights(cfg, dtype="f32")
        store = Q.ChunkStore(tmp_path / f"s{case}", cfg, dtype="f32")
        eng = Q.FusionEngine(w, store)
        ids, toks = [], []
        for _ in range(int(rng.integers(2, 5))):
            t = [int(x) for x in rng.integers(0, 256, int(rng.integers(16, 65)))]
            toks.append(t)
            ids.append(store.precompute(w, t, 0.05, "c").chunk_id)
        query = [int(x) for x in rng.integers(0, 256, int(rng.integers(4, 17)))]
        res = eng.run("QCFuse", 1.0, ids, query, max_new=32)
        fused = eng.assemble_context(ids)
        oracle = eng.oracle_run(fused.token_ids, query, max_new=32)
        div = float(np.abs(res.first_logits - oracle["first_logits"]).max())
        assert div < 1e-4, f"case {case}: logit divergence {div}"
        assert res.answer_tokens == oracle["answer_tokens"], f"case {case}: greedy mismatch"
        ow = O.init_weights(O.Config(seed=3000 + case))
        cpu = O.full_prefill_logits(ow, O.Fused(np.concatenate([np.asarray(t) for t in toks]), [], [], [], 0), query)
        assert np.abs(res.first_logits - cpu).max() < 1e-4, f"case {case}: vs CPU oracle"
    elapsed = time.time() - started
    assert elapsed < 60.0, f"took {elapsed:.1f} s"


def test_calibrate_layer_matches_reference_golden(golden_dir, tmp_path):
    """calibrate_layer (reference bench.py:118-144) on the chunks the reference
    retrieved for each query (tests/golden/calibrate.npz, made by running the
    reference): same per-layer mean overlaps and the same recommended layer."""
    import json

    import paper_2604_08585_b200 as Q
    from paper_2604_08585_b200.calibrate import calibrate_layer
    z = np.load(golden_dir / "calibrate.npz")
    d = json.loads(str(z["cfg"]))
    cfg = Q.ModelConfig(**{k: d[k] for k in ("n_layers", "n_heads", "d_model", "d_head", "d_ff", "rope_theta",
                                              "ln_eps", "seed", "critical_layer")})
    w = Q.init_weights(cfg, dtype="f32")
    store = Q.ChunkStore(tmp_path, cfg, dtype="f32", persist=False)
    for i in range(int(z["n_texts"])):
        store.precompute(w, z[f"text{i}_tokens"], 0.05, f"t{i}")
    eng = Q.FusionEngine(w, store)
    lists, queries = [], []
    for qi in range(int(z["n_queries"])):
        lists.append([Q.chunk_hash(z[f"query{qi}_chunk{ci}_tokens"]) for ci in range(int(z["top_k"]))])
        queries.append(z[f"query{qi}"].tolist())
    res = calibrate_layer(eng, lists, queries, ratio=float(z["ratio"]))
    got = np.asarray([res["mean_overlap"][int(l)] for l in z["layers"]])
    assert np.allclose(got, z["mean_overlap"], atol=1e-12), (got, z["mean_overlap"])
    assert res["recommended"] == int(z["recommended"])


@pytest.mark.parametrize("dtype,scoring", [("f32", "native"), ("bf16", "native"), ("bf16", "fp32")])
def test_ragged_batch_equals_single_requests(tmp_path, dtype, scoring):
    """A RAGGED batch (different chunk counts and lengths, query lengths and
    hence selection sizes) runs as one padded layer stack and gives
    every request what it gets alone: f32 bit-exact; bf16 against the oracle
    within the stated tolerance is covered per request by
    test_gpu_bf16_parity.py, here selection and logits track the single-request
    run (the fp32-scoring selection bit-exactly)."""
    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=4, d_model=512, d_head=128, d_ff=1024, seed=98)
    w = Q.init_weights(cfg, dtype=dtype, scoring=scoring)
    store = Q.ChunkStore(tmp_path / "s", cfg, dtype=dtype, persist=False, scoring=scoring)
    eng = Q.FusionEngine(w, store)
    lens = [96, 64, 130, 96, 48, 200, 96]
    pool = [store.precompute(w, np.random.default_rng(i).integers(0, 256, n), 0.05).chunk_id
            for i, n in enumerate(lens)]
    rng = np.random.default_rng(4)
    reqs = [[pool[j] for j in rng.permutation(len(pool))[:k]] for k in (3, 1, 4, 2, 3)]
    queries = [rng.integers(0, 256, n).tolist() for n in (12, 5, 20, 1, 12)]
    for use_graph in (False, True):
        plans, b = eng.prefill_batch("QCFuse", 0.2, reqs, queries, use_graph=use_graph)
        assert b.ragged
        for r in range(len(reqs)):
            logits, sel = eng.fuse(queries[r], reqs[r], 0.2)
            bsel = b.selection(r).cpu().numpy()
            blog = b.logits[r].cpu().numpy()
            assert bsel.size == plans[r].n_sel
            if dtype == "f32" or scoring == "fp32":
                assert np.array_equal(bsel, sel), r
            if dtype == "f32":
                assert np.array_equal(blog, logits), r
            else:
                assert len(set(bsel.tolist()) & set(sel.tolist())) >= 0.95 * sel.size
                assert np.abs(blog - logits).max() < 2e-2 * np.abs(logits).max()
    # the public batched entry returns each request's own selection
    lg, sels = eng.fuse_batch(queries, reqs, 0.2)
    assert [s.size for s in sels] == [p.n_sel for p in plans]


def test_batching_frontend_concurrent_threads(tmp_path):
    """Concurrent Python threads (the reference's FastAPI pattern) submit to the
    dynamic batcher: requests of different shapes are served in shared ragged
    batches, and each caller gets exactly what fuse() gives its request alone
    (f32 parity mode: bit-exact)."""
    from concurrent.futures import ThreadPoolExecutor

    import paper_2604_08585_b200 as Q
    cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=64, d_head=32, d_ff=128, seed=21)
    w = Q.init_weights(cfg, dtype="f32")
    store = Q.ChunkStore(tmp_path / "s", cfg, dtype="f32", persist=False)
    eng = Q.FusionEngine(w, store)
    pool = [store.precompute(w, np.random.default_rng(i).integers(0, 256, 24 + 8 * i), 0.1).chunk_id
            for i in range(6)]
    rng = np.random.default_rng(7)
    reqs = [([pool[j] for j in rng.permutation(6)[:int(rng.integers(1, 4))]],
             rng.integers(0, 256, int(rng.integers(2, 9))).tolist()) for _ in range(16)]
    alone = [eng.fuse(q, ids, 0.25) for ids, q in reqs]
    with Q.BatchingFrontend(eng, max_batch=8, max_wait_ms=20.0) as fe:
        with ThreadPoolExecutor(16) as pool_ex:
            futs = [pool_ex.submit(fe.fuse, q, ids, 0.25) for ids, q in reqs]
            got = [f.result() for f in futs]
        assert sum(fe.batches) == 16 and len(fe.batches) < 16
        with pytest.raises(KeyError):
            fe.submit([1, 2], ["ab" * 32])
    for (l0, s0), (l1, s1) in zip(alone, got):
        assert np.array_equal(s0, s1) and np.array_equal(l0, l1)


def test_sharded_pool_p2p(tmp_path):
    """ShardedChunkStore: two ranks each own half of the
    chunk pool and map the other's through CUDA IPC; fused prefills that draw
    chunks from both shards read the peer's HBM in place and equal a local pool
    bit for bit, and the oracle on the same chunk KV (selection bit-exact,
    logits 1e-4). Both ranks share this box's one GPU here (the same IPC path
    a multi-GPU node uses over NVLink)."""
    import json
    import socket
    import subprocess
    import sys
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    worker = str(Path(__file__).resolve().parent / "sharded_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), "2", str(port), str(tmp_path)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    for r in range(2):
        rep = json.loads((tmp_path / f"rank{r}.json").read_text())
        assert rep["remote"] > 0 and rep["owners"] == [0, 1]
        assert any(c["remote_chunks"] > 0 for c in rep["cases"])
        for c in rep["cases"]:
            assert c["equal_local"] and c["sel_equal_oracle"] and c["logit_err"] < 1e-4, c
        assert rep["batch_equal_local"]


class TestFetchLayer:
    """The reference's TestFetchLayer (test_store.py:149-199) against the B200
    store (f32 pool: the returned HostLayerKV is the device pool read back)."""

    @staticmethod
    def _store(tmp_path, **kw):
        import paper_2604_08585_b200 as Q
        cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234)
        return Q, cfg, Q.init_weights(cfg, dtype="f32"), Q.ChunkStore(tmp_path / "s", cfg, dtype="f32", **kw)

    def test_duration_formula(self, tmp_path):
        import paper_2604_08585_b200 as Q
        cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=16, d_head=8, d_ff=32, seed=3)
        store = Q.ChunkStore(tmp_path / "s", cfg, dtype="f32",
                             tier=Q.TierConfig(ssd_base_latency=0.001, ssd_bandwidth=1e6))
        rec = store.precompute(Q.init_weights(cfg, dtype="f32"), list(range(8)))
        _, duration = store.fetch_layer(rec.chunk_id, 1)
        assert duration == pytest.approx(0.001 + 1024 / 1e6)

    def test_counters_and_determinism(self, tmp_path):
        Q, cfg, w, store = self._store(tmp_path)
        rec = store.precompute(w, [5, 6, 7, 8])
        f0, b0 = store.manifest.layers_fetched, store.manifest.bytes_fetched
        kv1, _ = store.fetch_layer(rec.chunk_id, 2)
        kv2, _ = store.fetch_layer(rec.chunk_id, 2)
        assert np.array_equal(kv1.keys, kv2.keys)
        assert store.manifest.layers_fetched - f0 == 2
        assert store.manifest.bytes_fetched - b0 == 2 * (2 * 4 * 2 * 16 * 4)
        # the layer is the device pool's layer (and the oracle's precompute to fp32 rounding)
        ow = O.init_weights(O.Config(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234))
        ref = O.precompute_chunk(ow, [5, 6, 7, 8], 0.05)
        assert np.array_equal(kv1.keys, rec.k[1].cpu().numpy())
        assert np.abs(kv1.keys - ref.kv[1].keys).max() < 1e-5
        assert np.abs(kv1.values - ref.kv[1].values).max() < 1e-5

    def test_clock_advances(self, tmp_path):
        import paper_2604_08585_b200 as Q
        clock = Q.store.VirtualClock()
        cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234)
        store = Q.ChunkStore(tmp_path / "s", cfg, dtype="f32", clock=clock)
        rec = store.precompute(Q.init_weights(cfg, dtype="f32"), [1])
        _, d = store.fetch_layer(rec.chunk_id, 1)
        assert clock.now == pytest.approx(d)

    def test_layer_out_of_range_and_unknown(self, tmp_path):
        Q, cfg, w, store = self._store(tmp_path)
        rec = store.precompute(w, [1, 2])
        for bad in (0, 5):
            with pytest.raises(KeyError):
                store.fetch_layer(rec.chunk_id, bad)
        with pytest.raises(KeyError):
            store.fetch_layer("ff" * 32, 1)

    def test_anchor_rows_free_when_resident(self, tmp_path):
        Q, cfg, w, store = self._store(tmp_path)
        rec = store.precompute(w, list(range(30)), anchor_ratio=0.2)
        k, v, idx, duration = store.fetch_anchor_rows(rec.chunk_id, 1)
        assert duration == 0.0
        assert np.array_equal(idx, rec.anchor_indices)
        assert np.array_equal(k, rec.layer_kv[0].keys[idx]) and np.array_equal(v, rec.layer_kv[0].values[idx])

    def test_anchor_rows_charged_when_not_resident(self, tmp_path):
        Q, cfg, w, store = self._store(tmp_path, tier=None)
        store.tier = Q.TierConfig(anchors_resident=False)
        rec = store.precompute(w, list(range(30)), anchor_ratio=0.2)
        *_, duration = store.fetch_anchor_rows(rec.chunk_id, 1)
        assert duration > 0


def test_host_pool_matches_oracle(tmp_path):
    """The pinned-host pool's layer-pipelined prefill against the ORACLE (not
    only against the HBM pool): f32 parity mode, chunks from the oracle's
    precompute; selection bit-exact, first-token logits within 1e-4."""
    import paper_2604_08585_b200 as Q
    from tests.gpu_util import device_weights
    oc = O.Config(n_layers=4, n_heads=2, d_model=64, d_head=32, d_ff=128, seed=44)
    ow = O.init_weights(oc)
    rng = np.random.default_rng(8)
    chunks = [O.precompute_chunk(ow, rng.integers(0, 256, 40), 0.1) for _ in range(3)]
    query = rng.integers(0, 256, 7).tolist()
    ref = O.run(ow, chunks, query, 0.25)
    w = device_weights(ow, "f32")
    host = Q.ChunkStore(tmp_path / "h", w.config, dtype="f32", persist=False, pool="host")
    ids = load_oracle_chunks(host, chunks)
    assert host.get_record(ids[0]).on_host
    lg, sel = Q.FusionEngine(w, host).fuse(query, ids, 0.25)
    assert np.array_equal(sel, ref.selection)
    assert np.abs(lg - ref.first_logits).max() < 1e-4
