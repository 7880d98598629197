"""Concurrency: several host threads issue pulls on their own CUDA streams
through ONE peer (kvd_pull is serialised by the peer's mutex, the kernels
run concurrently, each request owns its completion slot), and two peers pull
into one decode cache at the same time.  Destinations are disjoint, so the
oracle applied in any order gives the expected bytes."""
import threading

import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, cache_for, make_pair, next_request_id

pytestmark = pytest.mark.gpu

G = kvdgen.CacheGeom(3, 4, 64, 16, 512, kvdgen.FP16)


def test_threads_and_streams_share_one_peer():
    pair = make_pair(G, G, seed=70)
    try:
        tables = kvdgen.disjoint_fragmented_tables([40] * 8, 512, 512, seed=4)
        ids = [[next_request_id() for _ in range(2)] for _ in range(4)]
        errors = []

        def worker(w):
            try:
                stream = torch.cuda.Stream()
                mine = tables[2 * w:2 * w + 2]
                for rid, (s, d) in zip(ids[w], mine):
                    pair.peer.pull(rid, s, d, stream)
                for rid in ids[w]:
                    pair.peer.wait(rid)
            except Exception as e:   # pragma: no cover - reported below
                errors.append(e)

        threads = [threading.Thread(target=worker, args=(w,)) for w in range(4)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errors, errors
        exp = pair.dst_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_two_peers_into_one_decode_cache():
    """Two prefill caches (e.g. two prefill workers) pulled concurrently into
    disjoint blocks of one decode cache, on two streams."""
    a = make_pair(G, G, seed=71)
    other = cache_for(G, 0)
    other_host = [kvdgen.random_bytes(other.layer_bytes, 9000 + l) for l in range(G.num_layers)]
    for t, h in zip(other.layers, other_host):
        t.copy_(torch.from_numpy(h))
    torch.cuda.synchronize()
    p2 = a.dst.open_peer(other.export())
    try:
        (s1, d1), (s2, d2) = kvdgen.disjoint_fragmented_tables([120, 130], 512, 512, seed=6)
        st1, st2 = torch.cuda.Stream(), torch.cuda.Stream()
        r1, r2 = next_request_id(), next_request_id()
        a.peer.pull(r1, s1, d1, st1)
        p2.pull(r2, s2, d2, st2)
        a.peer.wait(r1)
        p2.wait(r2)
        exp = a.expected(s1, d1)
        from oracle import oracle
        rc = oracle.pull(other_host, G.stride, G.num_blocks, exp, G.stride, G.num_blocks,
                         G.num_kv_heads, G.head_dim, G.block_size, G.elem_bytes, s2, d2)
        assert rc == oracle.OK
        assert_layers_equal(a.download_dst(), exp)
        # each exporter hears only about its own requests
        assert a.src.poll_released() == [r1]
        assert other.poll_released() == [r2]
    finally:
        p2.close()
        other.close()
        a.close()


def test_slot_exhaustion_and_recovery():
    """1024 completion slots per peer: more un-polled requests than slots is
    KVD_EBUSY, polling frees them."""
    from paper_2501_14743_b200 import kvd
    pair = make_pair(kvdgen.C1, kvdgen.C1, seed=72)
    try:
        rids = []
        with pytest.raises(kvd.KvdError) as ei:
            for _ in range(1100):
                rid = next_request_id()
                pair.peer.pull(rid, [], [])
                rids.append(rid)
        assert ei.value.status == kvd.EBUSY and len(rids) == 1024
        for r in rids:
            pair.peer.wait(r)
        rid = next_request_id()
        pair.peer.pull(rid, [1], [2])
        pair.peer.wait(rid)
    finally:
        pair.close()


def test_library_streams_overlap_and_order():
    """KVD_OPT_STREAMS = 2: transfers fork off the caller's stream (after the
    work already queued there) onto library streams; kvd_stream_wait joins
    them back.  Bytes stay the oracle's."""
    from paper_2501_14743_b200 import kvd
    pair = make_pair(G, G, seed=73)
    try:
        pair.peer.set(kvd.OPT_STREAMS, 2)
        user = torch.cuda.Stream()
        tables = kvdgen.disjoint_fragmented_tables([40, 33, 51, 20, 64], 512, 512, seed=7)
        zero_host = [np.zeros_like(h) for h in pair.dst_host]
        with torch.cuda.stream(user):
            torch.cuda._sleep(200_000_000)                 # ~0.1 s: the pulls must wait for it
            for t in pair.dst.layers:
                t.zero_()                                   # ... and for this fill
        rids = []
        for s, d in tables:
            rid = next_request_id()
            pair.peer.pull(rid, s, d, user)
            rids.append(rid)
        pair.peer.stream_wait(user)                         # user stream after every pull
        with torch.cuda.stream(user):
            got = [t.clone() for t in pair.dst.layers]      # read on the user stream, no host poll
        user.synchronize()
        exp = zero_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal([g.cpu().numpy() for g in got], exp)
        for rid in rids:
            pair.peer.wait(rid)
        assert sorted(pair.src.poll_released()) == sorted(rids)   # completion order may vary
        pair.peer.set(kvd.OPT_STREAMS, 0)                   # back to stream order
        s, d = kvdgen.disjoint_fragmented_tables([10], 512, 512, seed=8)[0]
        rid = next_request_id()
        pair.peer.pull(rid, s, d, user)
        pair.peer.wait(rid)
    finally:
        pair.close()


def test_poll_many_retires_completed_requests():
    """kvd_poll_many: one call reports (and retires) every completed request."""
    from paper_2501_14743_b200 import kvd
    pair = make_pair(G, G, seed=74)
    try:
        tables = kvdgen.disjoint_fragmented_tables([30, 45, 12, 60, 7], 512, 512, seed=9)
        rids = []
        for s, d in tables:
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            rids.append(rid)
        pending, seen = list(rids), []
        while pending:
            got = pair.peer.poll_many(pending)
            seen += got
            pending = [r for r in pending if r not in got]
        assert sorted(seen) == sorted(rids)
        with pytest.raises(kvd.KvdError) as ei:          # retired ids are no longer in flight
            pair.peer.poll_many(rids[:1])
        assert ei.value.status == kvd.EINVAL
        assert pair.peer.poll_many([]) == []
        exp = pair.dst_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()
