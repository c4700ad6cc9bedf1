"""B200-native QCFuse cache-fusion engine (arxiv 2604.08585) behind the
reference package's Python API. The compute path is the sm_100a C-ABI library
`libqcfuse_b200.so`; importing the engine fails loudly when it is missing."""

from .model import (BOS_ID, EOS_ID, PAD_ID, VOCAB_SIZE, ModelConfig, ModelWeights, byte_tokens,
                    init_weights, render_tokens, tokenize)
from .store import ChunkRecord, ChunkStore, FingerprintMismatch, StoreError, TierConfig, chunk_hash, extract_anchors
from .fusion import (POLICIES, PROBE_ANCHORS, PROBE_FULL, PROBE_NONE, FusedContext, FusionEngine,
                     QueryProbe, RecomputeTrace, RunOptions, RunResult, SelectionResult, select_topn,
                     sparse_attention, top_n_positions)
from .pipeline import CostModel
from .calibrate import calibrate_layer, layer_overlaps
from .serving import BatchingFrontend
from .sharded import ShardedChunkStore

__all__ = [n for n in dir() if not n.startswith("_")]
