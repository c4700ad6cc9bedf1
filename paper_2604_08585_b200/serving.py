"""Concurrent request front end: dynamic batching over the fused path.

The reference serves `FusionEngine.run` from FastAPI's thread pool and claims
engine re-entrancy (fusion.py:211-216). On the B200, running
concurrent requests as separate small launches on separate streams leaves the
tensor cores underfed (one request is ~800 recompute rows). Concurrent callers
therefore submit to a queue. One worker thread drains it into ragged batches,
up to `max_batch` requests or `max_wait_ms` after the first arrival, and runs
each batch as ONE fused prefill (`FusionEngine.fuse_batch`: one layer stack
over every request's rows, see fusion._Bufs). Each caller gets its own request's
first-token logits and selection through a Future, and every request's results
equal what `fuse()` gives it alone.
"""

from __future__ import annotations

import queue
import threading
import time
from concurrent.futures import Future
from dataclasses import dataclass

from .fusion import FusionEngine


@dataclass
class _Req:
    query: list
    chunk_ids: list
    ratio: float
    fut: Future


class BatchingFrontend:
    """Thread-safe `submit(query, chunk_ids, ratio) -> Future[(logits, selection)]`."""

    def __init__(self, engine: FusionEngine, max_batch: int = 8, max_wait_ms: float = 2.0):
        if max_batch < 1:
            raise ValueError("max_batch must be >= 1")
        self.engine = engine
        self.max_batch = max_batch
        self.max_wait = max_wait_ms / 1e3
        self._q: "queue.Queue[_Req | None]" = queue.Queue()
        self._closed = False
        self.batches: list[int] = []        # sizes of the batches run (observability)
        self._worker = threading.Thread(target=self._loop, name="qcf-batcher", daemon=True)
        self._worker.start()

    def submit(self, query, chunk_ids, ratio: float = 0.15) -> Future:
        if self._closed:
            raise RuntimeError("front end is closed")
        if not (0.0 <= ratio <= 1.0):
            raise ValueError("ratio must be in [0, 1]")
        qt = list(query.encode("utf-8")) if isinstance(query, str) else list(query)
        if not qt:
            raise ValueError("query must be non-empty")
        if not chunk_ids:
            raise ValueError("chunk list must be non-empty")
        for cid in chunk_ids:   # a bad request fails alone, before it can join a batch
            if cid not in self.engine.store:
                raise KeyError(f"unknown chunk: {cid}")
        fut: Future = Future()
        self._q.put(_Req(qt, list(chunk_ids), float(ratio), fut))
        return fut

    def fuse(self, query, chunk_ids, ratio: float = 0.15):
        """Blocking form of submit()."""
        return self.submit(query, chunk_ids, ratio).result()

    def close(self) -> None:
        if not self._closed:
            self._closed = True
            self._q.put(None)
            self._worker.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------
    def _loop(self) -> None:
        stop = False
        while not stop:
            first = self._q.get()
            if first is None:
                break
            batch = [first]
            deadline = time.perf_counter() + self.max_wait
            while len(batch) < self.max_batch:
                left = deadline - time.perf_counter()
                if left <= 0:
                    break
                try:
                    nxt = self._q.get(timeout=left)
                except queue.Empty:
                    break
                if nxt is None:
                    stop = True
                    break
                batch.append(nxt)
            # one prefill per ratio (the batched launch takes one recompute ratio)
            by_ratio: dict[float, list[_Req]] = {}
            for r in batch:
                by_ratio.setdefault(r.ratio, []).append(r)
            for ratio, reqs in by_ratio.items():
                self._run(ratio, reqs)

    def _run(self, ratio: float, reqs: list[_Req]) -> None:
        try:
            logits, sels = self.engine.fuse_batch([r.query for r in reqs], [r.chunk_ids for r in reqs], ratio)
        except Exception as e:   # a bad request fails its batch; report to every caller
            for r in reqs:
                r.fut.set_exception(e)
            return
        self.batches.append(len(reqs))
        for i, r in enumerate(reqs):
            r.fut.set_result((logits[i], sels[i]))
