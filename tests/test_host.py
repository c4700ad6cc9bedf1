"""CPU tests (no GPU): the C-ABI library loads and exports every declared
symbol; the host-side logic (store format, manifest, selection helpers, cost
model, request sharding) matches the reference's behaviour."""

import json
import re
import shutil
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "qcfuse_b200.h").read_text()
    return sorted(set(re.findall(r"\b(qcf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2604_08585_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(_lib.lib, s), s
        assert s in _lib.SIGNATURES, f"{s} declared in the header but not bound"
    assert set(_lib.SIGNATURES) == set(syms)
    assert _lib.lib.qcf_version().startswith(b"qcfuse_b200")


def test_library_is_sm100a():
    import subprocess
    so = ROOT / "paper_2604_08585_b200" / "libqcfuse_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_map_to_reference_exceptions():
    from paper_2604_08585_b200 import _lib
    with pytest.raises(ValueError):
        _lib.call("qcf_topn", None, 10, 3, 1, None, None, 0, None)
    with pytest.raises(ValueError):
        _lib.call("qcf_gemm", 0, None, 1, None, 1, None, 1, 1, 1, 1, 0, 0, None)


def test_qcfk_reads_reference_written_file(tmp_path, golden_dir):
    from paper_2604_08585_b200.model import ModelConfig
    from paper_2604_08585_b200.store import (config_fingerprint, read_qcfk, write_qcfk, chunk_hash,
                                              Manifest)
    host = json.loads((golden_dir / "host_logic.json").read_text())
    cfg = ModelConfig(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234)
    assert config_fingerprint(cfg) == host["fingerprint"]
    src = golden_dir / "ref_store"
    man = Manifest.loads((src / "manifest.txt").read_text())
    assert man.fingerprint == host["fingerprint"]
    rel = man.chunks[host["chunk_id"]][0]
    toks, k, v, norms, anchors, name = read_qcfk(src / rel, host["fingerprint"])
    assert chunk_hash(toks) == host["chunk_id"]
    assert anchors.tolist() == host["anchors"] and name == "ref-chunk"
    assert k.shape == (4, 19, 2, 16)
    # byte-identical rewrite (format parity, store.py:134-155)
    out = tmp_path / "x.qcfk"
    write_qcfk(out, host["fingerprint"], toks, k, v, norms, anchors, name)
    assert out.read_bytes() == (src / rel).read_bytes()


def test_qcfk_corruption_and_fingerprint(tmp_path, golden_dir):
    from paper_2604_08585_b200.store import FingerprintMismatch, StoreError, read_qcfk
    host = json.loads((golden_dir / "host_logic.json").read_text())
    src = next((golden_dir / "ref_store").rglob("*.qcfk"))
    raw = src.read_bytes()
    bad = tmp_path / "bad.qcfk"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(StoreError):
        read_qcfk(bad, None)
    bad.write_bytes(raw[:-3])
    with pytest.raises(StoreError):
        read_qcfk(bad, None)
    with pytest.raises(FingerprintMismatch):
        read_qcfk(src, "00" * 32)


def test_store_opens_reference_store_and_rejects_other_config(tmp_path, golden_dir):
    from paper_2604_08585_b200.model import ModelConfig
    from paper_2604_08585_b200.store import ChunkStore, FingerprintMismatch
    root = tmp_path / "s"
    shutil.copytree(golden_dir / "ref_store", root)
    cfg = ModelConfig(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64, seed=1234)
    st = ChunkStore(root, cfg, dtype="f32", device="cpu")
    host = json.loads((golden_dir / "host_logic.json").read_text())
    assert host["chunk_id"] in st
    rec = st.get_record(host["chunk_id"])          # device="cpu" here: pool on host for the test
    assert rec.n_tokens == 19 and rec.anchor_indices.tolist() == host["anchors"]
    with pytest.raises(KeyError):
        st.get_record("ab" * 32)
    with pytest.raises(FingerprintMismatch):
        ChunkStore(root, ModelConfig(seed=99), device="cpu")


def test_extract_anchors_rules():
    from paper_2604_08585_b200.store import extract_anchors
    assert extract_anchors([3.0, 1.0, 2.0], 1 / 3).tolist() == [0]
    assert extract_anchors([1.0, 1.0], 0.5).tolist() == [0]
    assert extract_anchors([0.5, 2.0, 1.0], 1.0).tolist() == [0, 1, 2]
    with pytest.raises(ValueError):
        extract_anchors([], 0.5)


def test_random_and_epic_select_match_reference(golden_dir):
    from paper_2604_08585_b200.fusion import epic_select, random_select, n_select
    host = json.loads((golden_dir / "host_logic.json").read_text())
    for key, idx in host["random_select"].items():
        seed, n, r = key.split("_")
        assert random_select(int(seed), int(n), float(r)).indices.tolist() == idx
    assert epic_select(40, 0.2, [(1, 15), (16, 25)]).indices.tolist() == host["epic"]
    assert n_select(0.07, 100) == 8          # ceil in double (fusion.py:155)
    with pytest.raises(ValueError):
        n_select(1.5, 10)


def test_cost_model_schedule_matches_reference(golden_dir):
    from paper_2604_08585_b200.model import ModelConfig
    from paper_2604_08585_b200.pipeline import CostModel, policy_schedule, schedule_pipelined
    host = json.loads((golden_dir / "host_logic.json").read_text())["schedule_qcfuse"]
    sch = policy_schedule("QCFuse", 51, 256, 16, ModelConfig(), CostModel())
    assert sch.ttft == host["ttft"] and sch.compute_end == host["compute_end"]
    assert schedule_pipelined([2, 2, 2], [3, 3, 3]).ttft == 11


def test_model_config_mirrors_reference():
    from paper_2604_08585_b200.model import ModelConfig, byte_tokens, tokenize
    assert ModelConfig().critical_layer == 2
    for bad in (dict(n_layers=3), dict(d_model=30), dict(critical_layer=1), dict(critical_layer=4),
                dict(vocab_size=300)):
        with pytest.raises(ValueError):
            ModelConfig(**bad)
    assert tokenize("Hi") == [256, 72, 105] and byte_tokens("Hi") == [72, 105]


def test_shard_blocks_cover_everything():
    from paper_2604_08585_b200.dist import shard
    for n in (0, 1, 7, 64, 65):
        for w in (1, 2, 3, 8):
            got = [i for r in range(w) for i in shard(n, w, r)]
            assert got == list(range(n))
            sizes = [len(shard(n, w, r)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def _gather_worker(rank, world, port, n_total, q):
    import os
    import torch.distributed as dist
    from paper_2604_08585_b200.dist import gather_rows, max_over_ranks, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(n_total, world, rank)
    local = torch.stack([torch.full((3,), float(i)) for i in mine]) if len(mine) else torch.zeros(0, 3)
    full = gather_rows(local, n_total, world, rank)
    t = max_over_ranks(float(rank + 1), "cpu")
    if rank == 0:
        q.put((full[:, 0].tolist(), t))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [5, 8])
def test_gather_two_ranks_gloo(n_total):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    rows, t = q.get()
    assert rows == [float(i) for i in range(n_total)]
    assert t == 2.0


def test_oracle_gqa_equals_mha_with_repeated_kv_weights():
    """The GQA restatement's semantics: a GQA model equals the MHA model whose
    wk/wv repeat each kv head's columns for the H/Hkv query heads sharing it."""
    from oracle import qcfuse_oracle as O
    g = O.Config(n_layers=4, n_heads=4, n_kv_heads=2, d_model=32, d_head=8, d_ff=64, seed=3)
    m = O.Config(n_layers=4, n_heads=4, d_model=32, d_head=8, d_ff=64, seed=3)
    wg = O.init_weights(g)
    layers = []
    for lw in wg.layers:
        rep = lambda w: np.repeat(w.reshape(32, 2, 8), 2, axis=1).reshape(32, 32)  # noqa: E731
        layers.append(O.Layer(lw.wq, rep(lw.wk), rep(lw.wv), lw.wo, lw.w1, lw.w2, lw.ln1_g, lw.ln1_b,
                              lw.ln2_g, lw.ln2_b))
    wm = O.Weights(m, wg.emb, layers, wg.lnf_g, wg.lnf_b)
    toks = np.random.default_rng(0).integers(0, 256, 21)
    a = O.forward_full(wg, toks, 0)
    b = O.forward_full(wm, toks, 0)
    assert np.allclose(a.logits, b.logits, atol=1e-6)
    assert np.array_equal(np.repeat(a.kv[2].keys, 2, axis=1), b.kv[2].keys)


def _bench_reference(env_extra, extra_args=(), drop=()):
    import os
    import subprocess
    import sys
    env = dict(os.environ, **env_extra)
    for k in drop:
        env.pop(k, None)
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "tiny",
                           "--steps", "1", "--warmup", "1", *extra_args], capture_output=True, text=True, env=env,
                          timeout=300)


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the CPU arm the driver times beside ours) prints
    one JSON line with the contract keys; warm-up is clamped to >= 3."""
    p = _bench_reference({"RANK": "0", "WORLD_SIZE": "1"})
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "requests/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_bench_reference_arm_other_ranks_exit_silently():
    p = _bench_reference({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, ["--gpus", "2"])
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_bench_reference_arm_reports_measured_and_extrapolated():
    p = _bench_reference({"RANK": "0", "WORLD_SIZE": "1"})
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["measured"]["layers"] == 4 and d["extrapolated"]["layers"] == 4
    # a step is the measured sample: steps x ms_per_step is time actually spent
    assert abs(d["ms_per_step"] - d["measured"]["ms_per_request_sample"]) < 1e-9
    assert d["host"]["cores"] >= 1 and d["host"]["cpu_model"]


def test_bench_gpus_flag_must_match_world():
    """--gpus N under a launcher with another WORLD_SIZE is an error, never a
    mislabelled line."""
    p = _bench_reference({"RANK": "0", "WORLD_SIZE": "1"}, ["--gpus", "2"])
    assert p.returncode != 0 and "WORLD_SIZE" in (p.stderr + p.stdout)


def test_bench_gpus_self_launches_n_ranks():
    """`python bench.py --gpus 2` (no launcher) re-executes itself under
    torch.distributed.run with 2 ranks on 127.0.0.1: rank 0 prints the line,
    rank 1 stays silent (the reference arm needs no GPU, so the spawn is
    exercised end to end on CPU)."""
    import bench
    cmd = bench.launch_cmd(2, ["--gpus", "2", "--steps", "1"])
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=2" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-4:] == ["--gpus", "2", "--steps", "1"]
    p = _bench_reference({}, ["--gpus", "2"], drop=("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"))
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference"


def test_batching_frontend_groups_and_routes_results():
    """Host logic of the dynamic batcher with a stand-in engine: concurrent
    submissions are grouped into batches of <= max_batch (split by ratio), each
    Future gets its own request's row, and a failing batch fails its callers."""
    import threading
    from concurrent.futures import ThreadPoolExecutor

    from paper_2604_08585_b200.serving import BatchingFrontend

    class FakeEngine:
        def __init__(self):
            self.store = {"a", "b", "c"}
            self.calls = []
            self.lock = threading.Lock()

        def fuse_batch(self, queries, chunk_lists, ratio):
            with self.lock:
                self.calls.append((len(queries), ratio))
            if any(q[0] == 255 for q in queries):
                raise ValueError("boom")
            return (np.asarray([[sum(q), ratio] for q in queries]),
                    [np.asarray([len(c)]) for c in chunk_lists])

    eng = FakeEngine()
    with BatchingFrontend(eng, max_batch=4, max_wait_ms=50.0) as fe:
        with ThreadPoolExecutor(10) as ex:
            futs = [ex.submit(fe.fuse, [i, 1], ["a"] * (1 + i % 3), 0.1 if i % 2 else 0.2) for i in range(10)]
            res = [f.result() for f in futs]
        for i, (lg, sel) in enumerate(res):
            assert lg.tolist() == [i + 1, 0.1 if i % 2 else 0.2] and sel.tolist() == [1 + i % 3]
        assert all(n <= 4 for n, _ in eng.calls) and sum(n for n, _ in eng.calls) == 10
        bad = fe.submit([255], ["a"])
        with pytest.raises(ValueError):
            bad.result(timeout=10)
        with pytest.raises(KeyError):
            fe.submit([1], ["zz"])
        with pytest.raises(ValueError):
            fe.submit([], ["a"])


def _sharded_worker(rank, world, port, root, q):
    import os
    import torch.distributed as dist
    import paper_2604_08585_b200 as Q
    from paper_2604_08585_b200.sharded import ShardedChunkStore
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=32, d_head=16, d_ff=64)
    st = ShardedChunkStore(Path(root) / f"r{rank}", cfg, dtype="f32", device="cpu")
    toks = [np.arange(5 + i) for i in range(10)]
    ids = []
    for t in toks:   # each rank registers only the chunks it owns (CPU tensors stand in for HBM)
        cid = Q.chunk_hash(t)
        ids.append(cid)
        if st.owner(cid) == rank:
            k = torch.full((4, t.size, 2, 16), float(int(cid[:4], 16)))
            st.add_record(t, k, -k, np.ones(t.size, np.float32), np.asarray([0]))
    st.exchange()
    res = []
    for cid in ids:
        rec = st.get_record(cid)
        res.append((cid, st.owner(cid), st.is_remote(cid), float(rec.k[0, 0, 0, 0]), float(rec.v[1, 0, 1, 2]),
                    tuple(rec.anchor_k.shape), rec.n_tokens))
    q.put((rank, res, sorted(st.chunk_ids()) == sorted(ids)))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_store_exchange_two_ranks_gloo(tmp_path):
    """ShardedChunkStore host logic over a 2-rank gloo group: every chunk has
    one owner, the exchange maps every peer chunk (metadata + shared tensors)
    into every rank, and a remote record reads the owner's values."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, str(tmp_path), q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get() for _ in range(2)]
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    by_rank = {r: res for r, res, _ in got}
    assert all(ok for _, _, ok in got)
    owners = {c[1] for c in by_rank[0]}
    assert owners == {0, 1}
    for rank, res in by_rank.items():
        for cid, owner, remote, kval, vval, ashape, n in res:
            assert remote == (owner != rank)
            assert kval == float(int(cid[:4], 16)) and vval == -kval
            assert ashape == (4, 1, 2, 16)
