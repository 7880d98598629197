"""The seeded input generators (kvdgen) produce valid, reproducible inputs
with the shapes the configs name (DESIGN.md §Input recipe)."""
import numpy as np
import pytest

import kvdgen


def _valid(src, dst, nb_s, nb_d):
    assert src.dtype == np.int32 and dst.dtype == np.int32 and src.shape == dst.shape
    assert len(set(dst.tolist())) == dst.size           # distinct destinations
    assert len(set(src.tolist())) == src.size           # a request owns distinct blocks
    assert (src >= 0).all() and (src < nb_s).all()
    assert (dst >= 0).all() and (dst < nb_d).all()


@pytest.mark.parametrize("n,nb", [(16, 64), (512, 1024), (1, 4), (100, 100)])
def test_fragmented_tables_valid_and_seeded(n, nb):
    a = kvdgen.fragmented_table(n, nb, nb, seed=1)
    b = kvdgen.fragmented_table(n, nb, nb, seed=1)
    _valid(*a, nb, nb)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_fragmented_run_statistics_c2():
    src, _ = kvdgen.fragmented_table(512, 1024, 1024, seed=1)
    runs = 1 + int(np.sum(np.diff(src) != 1))
    mean = 512 / runs
    assert 4 <= mean <= 16          # Geometric(mean 8), capped at 64


@pytest.mark.parametrize("run", [1, 2, 4, 8, 16, 32, 64])
def test_fixed_run_tables_do_not_merge_by_accident(run):
    n = 512
    src, dst = kvdgen.fixed_run_table(n, run, 2 * n + 64, 2 * n + 64, seed=5)
    _valid(src, dst, 2 * n + 64, 2 * n + 64)
    brk_s = np.flatnonzero(np.diff(src) != 1)
    # a break every `run` blocks exactly on both sides
    assert brk_s.size == -(-n // run) - 1
    assert np.all((brk_s + 1) % run == 0)


def test_mixed_requests_c3():
    toks = kvdgen.mixed_request_tokens(64, seed=0)
    assert len(toks) == 64 and min(toks) >= 512 and max(toks) <= 8192
    counts = [kvdgen.blocks_for(t, 16) for t in toks]
    tables = kvdgen.disjoint_fragmented_tables(counts, 2 * sum(counts), 2 * sum(counts), seed=3)
    all_dst = np.concatenate([t[1] for t in tables])
    assert len(set(all_dst.tolist())) == all_dst.size


def test_random_bytes_cover_all_words():
    words = kvdgen.random_bytes(1 << 22, seed=0).view(np.uint16)
    assert np.unique(words).size > 60000


def test_pattern_bytes_deterministic():
    a = kvdgen.pattern_bytes(4096, 1, 0, 3)
    assert np.array_equal(a, kvdgen.pattern_bytes(4096, 1, 0, 3))
    assert not np.array_equal(a, kvdgen.pattern_bytes(4096, 1, 1, 3))
