"""Pin the CPU oracle (oracle/qcfuse_oracle.py) to the reference.

Golden vectors come from `tests/golden/make_golden.py`, which ran the reference
package itself; the known-answer vectors are the reference's own
(`tests/test_model.py:28`, `tests/data/golden_logits_ab.json`,
`tests/test_fusion.py:168-170`, `tests/test_store.py:48-55`).
"""

import hashlib
from pathlib import Path
import json

import numpy as np
import pytest

from oracle import qcfuse_oracle as O

SM64_SEED0 = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def load_case(golden_dir, name):
    z = np.load(golden_dir / f"{name}.npz")
    cfgd = json.loads(str(z["cfg"]))
    cfg = O.Config(**{k: cfgd[k] for k in ("n_layers", "n_heads", "d_model", "d_head",
                                           "d_ff", "rope_theta", "ln_eps", "seed",
                                           "critical_layer")})
    n_chunks = len([k for k in z.files if k.endswith("_tokens") and k.startswith("chunk")])
    return z, cfg, n_chunks


class TestKnownAnswers:
    def test_splitmix64_seed0(self):
        assert [int(x) for x in O.splitmix64_at(0, np.arange(3))] == SM64_SEED0

    def test_uniform_top53(self):
        assert O.u64_to_unit(np.uint64((1 << 64) - 1)) == (2 ** 53 - 1) * 2.0 ** -53

    def test_golden_logits_ab(self, golden_dir):
        g = json.loads((golden_dir / "ref_golden_logits_ab.json").read_text())
        cfg = O.Config(n_layers=4, n_heads=2, d_model=16, d_head=8, d_ff=32, seed=7)
        lg = O.forward_full(O.init_weights(cfg), [O.BOS_ID] + list(b"ab")).logits
        assert lg.shape == tuple(g["shape"])
        got = lg[np.array(g["rows"]), np.array(g["cols"])]
        assert np.allclose(got, np.array(g["values"], np.float32), atol=1e-6)
        assert abs(float(lg.sum()) - g["checksum"]) < 1e-2

    def test_select_topn_example(self):
        assert O.select_topn([0.9, 0.1, 0.5, 0.4], 0.5).tolist() == [1, 3]

    def test_extract_anchors_examples(self):
        assert O.extract_anchors([3.0, 1.0, 2.0], 1 / 3).tolist() == [0]
        assert O.extract_anchors([1.0, 1.0], 0.5).tolist() == [0]

    def test_chunk_hash_vectors(self):
        assert O.chunk_hash([]) == hashlib.sha256(b"").hexdigest()
        toks = [81, 0, 65535]
        assert O.chunk_hash(toks) == hashlib.sha256(
            b"".join(t.to_bytes(4, "little") for t in toks)).hexdigest()

    def test_llama_width_init_draws(self, golden_dir):
        z = np.load(golden_dir / "init_llama_probe.npz")
        got = O.draw_uniform_f32(1234, 0, 1)
        assert got[0] == z["values"][0]
        for s, v in zip(z["steps"][::7], z["values"][::7]):
            assert O.draw_uniform_f32(1234, int(s), 1)[0] == v


@pytest.mark.parametrize("name", ["small_case0", "small_case1", "small_case2",
                                  "tiny_case0", "tiny_case1", "tiny_case2",
                                  "tiny_case3", "tiny_case4", "tiny_case5"])
def test_fused_path_matches_reference(golden_dir, name):
    z, cfg, nc = load_case(golden_dir, name)
    w = O.init_weights(cfg)
    chunks = [O.precompute_chunk(w, z[f"chunk{i}_tokens"], float(z["anchor_ratio"]))
              for i in range(nc)]
    for i, c in enumerate(chunks):
        assert np.array_equal(c.anchors, z[f"chunk{i}_anchors"])
        assert np.abs(c.key_norms - z[f"chunk{i}_norms"]).max() < 1e-5
    out = O.run(w, chunks, z["query"], float(z["ratio"]))
    assert out.fused.offsets == z["offsets"].tolist()
    rows = z["sample_rows"]
    full_rows = z["fused_k0"].shape[0] == out.fused.n_ctx + 1
    for li in range(cfg.n_layers):
        fk = out.fused.keys[li] if full_rows else out.fused.keys[li][rows]
        fv = out.fused.values[li] if full_rows else out.fused.values[li][rows]
        assert np.abs(fk - z[f"fused_k{li}"]).max() < 1e-5
        assert np.abs(fv - z[f"fused_v{li}"]).max() < 1e-5
    c = cfg.critical_layer
    assert np.array_equal(out.probe.prefix_positions, z["prefix_positions"])
    assert np.abs(out.probe.queries[c - 1] - z["q_c"]).max() < 1e-4
    assert np.abs(out.scores - z["scores"]).max() < 1e-6
    assert np.array_equal(out.selection, z["selection"])          # bit-exact index set
    assert np.abs(out.first_logits - z["first_logits"]).max() < 1e-4
    for li in range(cfg.n_layers):
        if full_rows:
            assert np.abs(out.updated.keys[li] - z[f"upd_k{li}"]).max() < 1e-4
            assert np.abs(out.updated.values[li] - z[f"upd_v{li}"]).max() < 1e-4
        else:
            r = z[f"upd_rows{li}"]
            assert np.abs(out.updated.keys[li][r] - z[f"upd_k{li}"]).max() < 1e-4
            assert np.abs(out.updated.values[li][r] - z[f"upd_v{li}"]).max() < 1e-4


def test_full_prefill_and_decode_match_reference(golden_dir):
    z, cfg, nc = load_case(golden_dir, "small_case0")
    w = O.init_weights(cfg)
    chunks = [O.precompute_chunk(w, z[f"chunk{i}_tokens"], float(z["anchor_ratio"]))
              for i in range(nc)]
    out = O.run(w, chunks, z["query"], float(z["ratio"]), max_new=8)
    assert out.answer == z["answer"].tolist()
    full = O.full_prefill_logits(w, out.fused, z["query"])
    assert np.abs(full - z["full_logits"]).max() < 1e-4


def test_ratio_one_equals_full_prefill(golden_dir):
    # fusion.py:302-307 equivalence, stated on the oracle
    z, cfg, nc = load_case(golden_dir, "small_case1")
    w = O.init_weights(cfg)
    chunks = [O.precompute_chunk(w, z[f"chunk{i}_tokens"], 0.05) for i in range(nc)]
    out = O.run(w, chunks, z["query"], 1.0)
    full = O.full_prefill_logits(w, out.fused, z["query"])
    assert np.abs(out.first_logits - full).max() < 1e-4


def _baseline_case(name):
    import json
    from oracle import qcfuse_oracle as O
    z = np.load(Path(__file__).parent / "golden" / "baselines.npz")
    d = json.loads(str(z[f"{name}_cfg"]))
    oc = O.Config(**{k: d[k] for k in ("n_layers", "n_heads", "d_model", "d_head", "d_ff", "rope_theta", "ln_eps",
                                       "seed", "critical_layer")})
    ow = O.init_weights(oc)
    chunks = [O.precompute_chunk(ow, z[f"{name}_chunk{i}_tokens"], 0.1) for i in range(int(z[f"{name}_n_chunks"]))]
    return z, oc, ow, chunks, O.assemble(ow, chunks)


@pytest.mark.parametrize("name", ["small", "small2", "tiny"])
def test_oracle_cacheblend_kvshare_vs_reference(name):
    """Oracle restatement of the layer-1 deviation policies reproduces the
    reference's deviations / received attention and its CacheBlend/KVShare
    index sets (fixtures by tests/golden/make_golden.py baselines)."""
    from oracle import qcfuse_oracle as O
    z, oc, ow, chunks, fused = _baseline_case(name)
    k, v, attn = O.layer1_recompute_pass(ow, fused)
    dev = O.kv_deviation(fused, k, v)
    assert np.allclose(dev, z[f"{name}_deviation"], rtol=1e-5)
    assert np.allclose(attn[:, :, 1:].mean(axis=(0, 1)), z[f"{name}_received"], rtol=1e-4, atol=1e-7)
    r = float(z[f"{name}_ratio"])
    assert np.array_equal(O.select_topn(O.cacheblend_scores(ow, fused), r), z[f"{name}_CacheBlend"])
    assert np.array_equal(O.select_topn(O.kvshare_scores(ow, fused), r), z[f"{name}_KVShare"])
