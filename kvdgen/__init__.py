"""kvdgen -- seeded synthetic inputs shared by the oracle tests, the GPU
parity tests and bench.py.

This module holds NO arithmetic of the method (no offsets, spans, runs or
copies): only the configurations of BASELINE.json (C1-C5), seeded block
tables shaped like a paged allocator's (contiguous, fragmented, worst case,
fixed run length, mixed request lengths) and seeded cache contents.  The
recipes are stated in DESIGN.md §"Input recipe".
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass, replace
from typing import List, Sequence, Tuple

import numpy as np

FP16, BF16, FP8, FP32 = 0, 1, 2, 3
ELEM_BYTES = {FP16: 2, BF16: 2, FP8: 1, FP32: 4}


@dataclass(frozen=True)
class CacheGeom:
    """One side's paged KV cache: one tensor per layer, Dims (B, KV, L, H, D)."""
    num_layers: int
    num_kv_heads: int       # per shard
    head_dim: int
    block_size: int         # tokens per block ("L" of Fig. 5)
    num_blocks: int         # "B" of Fig. 5
    dtype: int = FP16
    stride: Tuple[int, int, int, int, int] = (0, 0, 0, 0, 0)  # all zero: Fig. 5 default

    @property
    def elem_bytes(self) -> int:
        return ELEM_BYTES[self.dtype]

    def with_blocks(self, nb: int) -> "CacheGeom":
        return replace(self, num_blocks=nb)

    @property
    def bytes_per_token(self) -> int:
        """K + V bytes of one token across all layers (config bookkeeping)."""
        return 2 * self.num_layers * self.num_kv_heads * self.head_dim * self.elem_bytes


# BASELINE.json configs (SURVEY.md §8 row d table).
C1 = CacheGeom(num_layers=2, num_kv_heads=2, head_dim=64, block_size=16, num_blocks=64,
               dtype=FP16)
C2 = CacheGeom(num_layers=32, num_kv_heads=32, head_dim=128, block_size=16,
               num_blocks=1024, dtype=FP16)
C4 = CacheGeom(num_layers=80, num_kv_heads=2, head_dim=128, block_size=16,
               num_blocks=1024, dtype=BF16)
C1_TOKENS = 256
C2_TOKENS = 8192
C4_TOKENS = 8192
C3_REQUESTS = 64
C3_TOKENS = (512, 8192)


def blocks_for(tokens: int, block_size: int) -> int:
    return -(-tokens // block_size)


# --------------------------------------------------------------------------
# block tables
# --------------------------------------------------------------------------

def contiguous_table(n: int, src_start: int = 0, dst_start: int = 0):
    return (np.arange(src_start, src_start + n, dtype=np.int32),
            np.arange(dst_start, dst_start + n, dtype=np.int32))


def _run_lengths(n: int, rng: random.Random, mean: float, cap: int) -> List[int]:
    """Run lengths ~ Geometric(mean) capped at ``cap`` until they sum to n."""
    p = 1.0 / mean
    out = []
    left = n
    while left > 0:
        u = rng.random()
        k = 1 + int(math.log(1.0 - u) / math.log(1.0 - p)) if p < 1.0 else 1
        k = max(1, min(k, cap, left))
        out.append(k)
        left -= k
    return out


def _place_runs(lengths: Sequence[int], num_blocks: int, rng: random.Random,
                min_gap: int = 1) -> List[int]:
    """Place runs at random free offsets in [0, num_blocks) with at least
    ``min_gap`` free blocks between neighbouring runs, then visit the runs in
    random order (a fragmented free list).  Returns the block id sequence."""
    n = sum(lengths)
    k = len(lengths)
    slack = num_blocks - n - min_gap * (k - 1)
    if slack < 0 and min_gap > 0 and num_blocks >= n:
        min_gap = 0                      # a full pool cannot keep gaps
        slack = num_blocks - n
    if slack < 0:
        raise ValueError(f"pool of {num_blocks} blocks too small for {n} blocks in {k} runs")
    cuts = sorted(rng.randint(0, slack) for _ in range(k))
    starts, pos, prev = [], 0, 0
    for j, length in enumerate(lengths):
        pos += cuts[j] - prev
        prev = cuts[j]
        starts.append(pos)
        pos += length + min_gap
    order = list(range(k))
    rng.shuffle(order)
    ids: List[int] = []
    for j in order:
        ids.extend(range(starts[j], starts[j] + lengths[j]))
    return ids


def fragmented_table(n: int, src_blocks: int, dst_blocks: int, seed: int,
                     mean_run: float = 8.0, cap: int = 64):
    """Fragmented allocator state: runs ~ Geometric(mean 8) capped at 64 at
    random free offsets, drawn independently for the source and destination
    side (SURVEY.md §8 row d, C2 'fragmented')."""
    rng = random.Random(seed)
    src = _place_runs(_run_lengths(n, rng, mean_run, cap), src_blocks, rng)
    dst = _place_runs(_run_lengths(n, rng, mean_run, cap), dst_blocks, rng)
    return np.asarray(src, dtype=np.int32), np.asarray(dst, dtype=np.int32)


def fixed_run_table(n: int, run: int, src_blocks: int, dst_blocks: int, seed: int):
    """Runs of exactly ``run`` blocks (last one ragged), non-adjacent on both
    sides so they cannot merge by accident (C5 sweep)."""
    rng = random.Random(seed)
    lengths = [run] * (n // run) + ([n % run] if n % run else [])
    src = _place_runs(lengths, src_blocks, rng)
    dst = _place_runs(lengths, dst_blocks, rng)
    return np.asarray(src, dtype=np.int32), np.asarray(dst, dtype=np.int32)


def random_table(n: int, src_blocks: int, dst_blocks: int, seed: int):
    """Uniformly random distinct ids on both sides (fully fragmented)."""
    rng = np.random.default_rng(seed)
    src = rng.choice(src_blocks, size=n, replace=False).astype(np.int32)
    dst = rng.choice(dst_blocks, size=n, replace=False).astype(np.int32)
    return src, dst


def mixed_request_tokens(count: int = C3_REQUESTS, seed: int = 0,
                         lo: int = C3_TOKENS[0], hi: int = C3_TOKENS[1]) -> List[int]:
    """C3: prompt lengths ~ U{lo..hi} (random.Random(seed))."""
    rng = random.Random(seed)
    return [rng.randint(lo, hi) for _ in range(count)]


def disjoint_fragmented_tables(block_counts: Sequence[int], src_blocks: int,
                               dst_blocks: int, seed: int, mean_run: float = 8.0,
                               cap: int = 64):
    """Block tables for several requests that share one pool per side: the
    pools are carved into disjoint, fragmented allocations (no block is
    owned by two requests)."""
    rng = random.Random(seed)
    total = sum(block_counts)
    src_all = _place_runs(_run_lengths(total, rng, mean_run, cap), src_blocks, rng)
    dst_all = _place_runs(_run_lengths(total, rng, mean_run, cap), dst_blocks, rng)
    out, pos = [], 0
    for c in block_counts:
        out.append((np.asarray(src_all[pos:pos + c], dtype=np.int32),
                    np.asarray(dst_all[pos:pos + c], dtype=np.int32)))
        pos += c
    return out


# --------------------------------------------------------------------------
# cache contents
# --------------------------------------------------------------------------

def random_bytes(nbytes: int, seed: int) -> np.ndarray:
    """Uniform random bytes: every 16-bit word pattern occurs, so fp16/bf16
    NaN payloads, +-Inf, -0 and subnormals are all present."""
    return np.random.default_rng(seed).integers(0, 256, size=nbytes, dtype=np.uint8)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def pattern_bytes(nbytes: int, seed: int, side: int, layer: int) -> np.ndarray:
    """Counter-based structured fill (after SPEC.md's payload_byte idea,
    S:L433-437): byte k of a layer buffer = low byte of
    splitmix64(seed, side, layer, k).  Lets a test localise misplacement."""
    with np.errstate(over="ignore"):
        key = np.uint64((seed * 0x100000001B3 + side * 0x1000193 + layer) & (2**64 - 1))
        k = np.arange(nbytes, dtype=np.uint64)
        return (_splitmix64(k ^ (key << np.uint64(20))) & np.uint64(0xFF)).astype(np.uint8)


def torch_fill_random_(tensor, seed: int):
    """Fill a torch uint8/int tensor (any device) with seeded random bytes
    using torch's own generator; used for caches too big to build on host."""
    import torch
    gen = torch.Generator(device=tensor.device)
    gen.manual_seed(seed)
    flat = tensor.view(torch.uint8).view(-1)
    chunk = 1 << 28
    for off in range(0, flat.numel(), chunk):
        part = flat[off:off + chunk]
        part.copy_(torch.randint(0, 256, part.shape, dtype=torch.uint8, device=tensor.device,
                                 generator=gen))
    return tensor
