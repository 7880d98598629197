"""Pins for the oracle's coalescing rule (§4.2).

Checked against the fig:queue example (tests/golden/fig_queue_merge.txt),
SPEC.md's "fully bi-contiguous request -> one K run and one V run" property
 and a brute-force characterisation of maximal runs that does not
reuse the oracle's greedy loop.
"""
import os
import random

import pytest

from oracle import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SHAPE = (12, 2, 16, 2, 128)   # Fig. 5 geometry with a few more blocks
STRIDE = oracle.default_strides(12, 16, 2, 128)


def _cases():
    with open(os.path.join(GOLDEN, "fig_queue_merge.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            _, name, *rest = line.split()
            arrow = rest.index("->")
            pairs = [tuple(int(x) for x in p.split(":")) for p in rest[:arrow]]
            yield name, pairs, int(rest[arrow + 1])


@pytest.mark.parametrize("name,pairs,want", list(_cases()))
def test_fig_queue_cases(name, pairs, want):
    src = [p[0] for p in pairs]
    dst = [p[1] for p in pairs]
    streams = oracle.read_transactions(1, SHAPE, STRIDE, SHAPE, STRIDE, 2, src, dst)
    for stream in streams:                       # K and V stream alike
        assert len(oracle.coalesce(stream)) == want, name


@pytest.mark.parametrize("n", [1, 2, 5, 12])
def test_fully_bicontiguous_is_two_reads_per_layer(n):
    """a fully bi-contiguous n-block request -> exactly 2 reads per
    layer (one K run, one V run) for the [B][KV][L][H][D] layout."""
    layers = 3
    streams = oracle.read_transactions(layers, SHAPE, STRIDE, SHAPE, STRIDE, 2,
                                       list(range(n)), list(range(12 - n, 12)))
    merged = [r for s in streams for r in oracle.coalesce(s)]
    assert len(merged) == 2 * layers
    span = 16 * 2 * 128 * 2
    assert all(r.size == n * span for r in merged)


def _byte_map(reads):
    m = {}
    for r in reads:
        for k in range(0, r.size, 256):          # 256 B granules are enough
            key = (r.layer, r.kv, r.remote + k)
            assert key not in m
            m[key] = r.local + k
    return m


def test_coalesce_bruteforce_random_tables():
    """>=10^3 random tables: the coalesced reads move the
    same remote->local byte map, every read is bi-contiguous by
    construction, no two neighbours could merge (maximal), order kept."""
    rng = random.Random(7)
    nb = 12
    span = 16 * 2 * 128 * 2
    for trial in range(1000):
        n = rng.randint(0, nb)
        if rng.random() < 0.5:
            src = rng.sample(range(nb), n)
            dst = rng.sample(range(nb), n)
        else:   # runs likely
            s0, d0 = rng.randint(0, nb - n), rng.randint(0, nb - n)
            src = list(range(s0, s0 + n))
            dst = list(range(d0, d0 + n))
            cut = rng.randint(0, n)
            dst = dst[cut:] + dst[:cut]
        streams = oracle.read_transactions(1, SHAPE, STRIDE, SHAPE, STRIDE, 2, src, dst)
        for stream in streams:
            merged = oracle.coalesce(stream)
            assert _byte_map(merged) == _byte_map(stream)
            # maximality: neighbours are not bi-contiguous
            for a, b in zip(merged, merged[1:]):
                assert not (a.remote + a.size == b.remote and a.local + a.size == b.local)
            # order preserved: concatenating the merged reads block by block
            # reproduces the original sequence
            rebuilt = []
            for r in merged:
                for k in range(r.size // span):
                    rebuilt.append((r.remote + k * span, r.local + k * span))
            assert rebuilt == [(r.remote, r.local) for r in stream]
            # brute-force run count: 1 + number of i with a break between i, i+1
            breaks = sum(1 for i in range(n - 1)
                         if not (src[i + 1] == src[i] + 1 and dst[i + 1] == dst[i] + 1))
            assert len(merged) == (0 if n == 0 else 1 + breaks)
