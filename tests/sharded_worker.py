"""Worker for tests/test_gpu_parity.py::test_sharded_pool_p2p (one process per
rank; oracle = checker only). Run: python tests/sharded_worker.py RANK WORLD PORT OUT_DIR"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(rank: int, world: int, port: int, out: Path) -> None:
    import paper_2604_08585_b200 as Q
    from oracle import qcfuse_oracle as O
    from paper_2604_08585_b200.sharded import ShardedChunkStore
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    n_dev = torch.cuda.device_count()
    torch.cuda.set_device(rank % n_dev)
    cfg = Q.ModelConfig(n_layers=4, n_heads=2, d_model=64, d_head=32, d_ff=128, seed=31)
    w = Q.init_weights(cfg, dtype="f32")
    toks = [np.random.default_rng(i).integers(0, 256, 20 + 4 * i) for i in range(8)]
    store = ShardedChunkStore(out / f"s{rank}", cfg, dtype="f32")
    ids = store.precompute_shard(w, toks, 0.1)
    store.exchange()
    eng = Q.FusionEngine(w, store)
    local = Q.ChunkStore(out / f"l{rank}", cfg, dtype="f32", persist=False)
    lids = [local.precompute(w, t, 0.1).chunk_id for t in toks]
    assert lids == ids
    leng = Q.FusionEngine(w, local)
    ow = O.init_weights(O.Config(n_layers=4, n_heads=2, d_model=64, d_head=32, d_ff=128, seed=31))
    rng = np.random.default_rng(100 + rank)
    report = {"rank": rank, "remote": sum(store.is_remote(c) for c in ids),
              "owners": sorted({store.owner(c) for c in ids}), "cases": []}
    for _ in range(6):
        pick = [ids[j] for j in rng.permutation(len(ids))[:4]]
        query = rng.integers(0, 256, 6).tolist()
        lg, sel = eng.fuse(query, pick, 0.3)
        lg_l, sel_l = leng.fuse(query, pick, 0.3)
        # oracle on the same chunk KV (the parity bridge): selection bit-exact, logits 1e-4
        chunks = []
        for cid in pick:
            rec = local.get_record(cid)
            k, v = rec.k.cpu().numpy(), rec.v.cpu().numpy()
            chunks.append(O.Chunk(rec.token_ids, [O.KV(k[i], v[i], np.arange(rec.n_tokens)) for i in range(4)],
                                  rec.key_norms, rec.anchor_indices))
        ref = O.run(ow, chunks, query, 0.3)
        report["cases"].append({
            "remote_chunks": sum(store.is_remote(c) for c in pick),
            "equal_local": bool(np.array_equal(lg, lg_l) and np.array_equal(sel, sel_l)),
            "sel_equal_oracle": bool(np.array_equal(sel, ref.selection)),
            "logit_err": float(np.abs(lg - ref.first_logits).max())})
    # a batch mixing local and remote chunks
    reqs = [[ids[j] for j in rng.permutation(len(ids))[:3]] for _ in range(3)]
    qs = [rng.integers(0, 256, 5).tolist() for _ in range(3)]
    bl, bs = eng.fuse_batch(qs, reqs, 0.3)
    ll, ls = leng.fuse_batch(qs, reqs, 0.3)
    report["batch_equal_local"] = bool(np.array_equal(bl, ll) and all(np.array_equal(a, b) for a, b in zip(bs, ls)))
    torch.cuda.synchronize()
    dist.barrier()
    (out / f"rank{rank}.json").write_text(json.dumps(report))
    dist.barrier()   # owners keep their chunks alive until every peer is done
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), Path(sys.argv[4]))
