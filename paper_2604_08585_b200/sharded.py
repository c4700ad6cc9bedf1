"""Chunk pool sharded over the GPUs of one node, read in place over NVLink
("a sharded chunk pool via NVLink P2P reads").

Each chunk lives in the HBM of exactly one rank, its owner. The owner is the
chunk's content hash (store.py:52-56) mod world size. After `exchange()`,
every rank has mapped every other rank's chunk tensors into its own address
space through CUDA IPC. The handles travel once, over the process group. The
fused path then reads a remote chunk exactly as it reads a local one: its
`qcf_chunk_desc` holds the peer pointer, and `qcf_assemble` (the RoPE
re-alignment + concat) loads the chunk KV straight from the owner's HBM over
NVLink. There is no staging copy and no collective on the data path. The
pool then holds world x one GPU's chunks, the same total a replicated pool
holds on one GPU. Results are bit-identical to a local pool, since the same
kernels read the same bytes.

The anchor rows and (fp32 scoring mode) the float32 critical-layer keys are
exported the same way. The probe's prefix assembly also reads them in place.
Assembly of a remote chunk loads its K/V over NVLink (~900 GB/s per GPU per
direction on NVSwitch), about 7x less bandwidth than local HBM. A request
that draws most of its chunks from peers is assembly-bound accordingly.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist
from torch.multiprocessing.reductions import reduce_tensor

from .store import DEFAULT_ANCHOR_RATIO, ChunkRecord, ChunkStore, chunk_hash


def _export(t: torch.Tensor | None):
    return None if t is None else reduce_tensor(t)


def _import(h):
    if h is None:
        return None
    fn, args = h
    return fn(*args)


class ShardedChunkStore(ChunkStore):
    """ChunkStore whose chunks are spread over the ranks of `group` (default:
    the world). `precompute_shard` builds the locally owned chunks, and
    `exchange` (collective) maps every rank's chunks into every rank."""

    def __init__(self, root, config, group=None, **kw):
        if kw.get("pool", "hbm") != "hbm":
            raise ValueError("a sharded pool lives in HBM")
        kw.setdefault("persist", False)
        super().__init__(root, config, **kw)
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self._remote: dict[str, ChunkRecord] = {}

    # -- placement ------------------------------------------------------------
    def owner(self, chunk_id: str) -> int:
        return int(chunk_id[:16], 16) % self.world

    def is_remote(self, chunk_id: str) -> bool:
        return chunk_id in self._remote

    def precompute_shard(self, weights, token_lists, anchor_ratio: float = DEFAULT_ANCHOR_RATIO,
                         source_names=None) -> list[str]:
        """Precompute (GPU) the chunks this rank owns; returns the ids of ALL
        chunks (every rank computes the same list from the content hashes)."""
        names = list(source_names) if source_names is not None else [""] * len(token_lists)
        ids = []
        for t, name in zip(token_lists, names):
            cid = chunk_hash(np.asarray(t, np.int64))
            ids.append(cid)
            if self.owner(cid) == self.rank and cid not in self._cache:
                self.precompute(weights, t, anchor_ratio, name)
        return ids

    def exchange(self) -> None:
        """Collective over the group: every rank publishes its chunks (metadata
        plus CUDA IPC handles of the K/V, anchor-row and fp32-scoring tensors)
        and maps every other rank's."""
        mine = []
        for cid, rec in self._cache.items():
            if self.owner(cid) != self.rank:
                continue
            ak, av = self.anchor_kv(rec)
            mine.append({"cid": cid, "tokens": rec.token_ids, "norms": rec.key_norms,
                         "anchors": rec.anchor_indices, "name": rec.source_name,
                         "k": _export(rec.k), "v": _export(rec.v), "ak": _export(ak), "av": _export(av),
                         "kc32": _export(rec.k_crit32), "ak32": _export(rec.anchor_k32),
                         "av32": _export(rec.anchor_v32)})
        got = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(got, mine, group=self.group)
        else:
            got = [mine]
        for r, items in enumerate(got):
            if r == self.rank:
                continue
            for it in items:
                rec = ChunkRecord(it["cid"], it["tokens"], _import(it["k"]), _import(it["v"]), it["norms"],
                                  it["anchors"], it["name"])
                rec.anchor_k, rec.anchor_v = _import(it["ak"]), _import(it["av"])
                rec.k_crit32, rec.anchor_k32, rec.anchor_v32 = (_import(it["kc32"]), _import(it["ak32"]),
                                                                _import(it["av32"]))
                self._remote[rec.chunk_id] = rec
                self.manifest.chunks[rec.chunk_id] = (f"rank{r}", rec.n_tokens, len(rec.anchor_indices),
                                                      rec.source_name)
        if self.world > 1:
            dist.barrier(group=self.group)   # every peer has mapped before anyone launches on them

    # -- reads ----------------------------------------------------------------
    def get_record(self, chunk_id: str, with_tensors: bool = True) -> ChunkRecord:
        rec = self._remote.get(chunk_id)
        if rec is not None:
            return rec
        return super().get_record(chunk_id, with_tensors)

    def load_meta(self, chunk_id: str) -> ChunkRecord:
        rec = self._remote.get(chunk_id)
        if rec is not None:
            return ChunkRecord(rec.chunk_id, rec.token_ids, None, None, rec.key_norms, rec.anchor_indices,
                               rec.source_name)
        return super().load_meta(chunk_id)

    def anchor_kv(self, rec: ChunkRecord):
        if rec.anchor_k is not None:
            return rec.anchor_k, rec.anchor_v
        return super().anchor_kv(rec)
