"""Concurrency: several host threads issue pulls on their own CUDA streams
through ONE peer (kvd_pull is serialised by the peer's mutex, the kernels
run concurrently, each request owns its completion slot), and two peers pull
into one decode cache at the same time.  Destinations are disjoint, so the
oracle applied in any order gives the expected bytes."""
import threading
import time

import numpy as np
import pytest
import torch

import kvdgen
from paper_2501_14743_b200 import kvd
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


def test_poll_many_bad_input_changes_nothing():
    """All or nothing (kvd_poll_many): a duplicate or unknown id is refused
    before any request is retired, so completions are never lost."""
    from paper_2501_14743_b200 import kvd
    pair = make_pair(G, G, seed=75)
    try:
        tables = kvdgen.disjoint_fragmented_tables([20, 25, 30], 512, 512, seed=10)
        rids = []
        for s, d in tables:
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            rids.append(rid)
        torch.cuda.synchronize()                        # all three have completed
        for bad in (rids + [rids[1]], rids + [next_request_id() + 10**9]):
            with pytest.raises(kvd.KvdError) as ei:
                pair.peer.poll_many(bad)
            assert ei.value.status == kvd.EINVAL
        # nothing was retired by the failed calls: every id still reports once
        assert sorted(pair.peer.poll_many(rids)) == sorted(rids)
        exp = pair.dst_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_poll_does_not_wait_for_a_concurrent_launch():
    """kvd_poll_done is lock-free (SURVEY §8 b threading): a
    thread polling an in-flight request of a peer while another thread
    issues host-heavy kvd_pulls on the SAME peer (60k uncoalesced blocks
    each: validation, planning, a run-table upload and the launch) sees a
    poll latency that does not track the kvd_pull call time."""
    import time
    from paper_2501_14743_b200 import kvd
    g = kvdgen.CacheGeom(1, 1, 64, 16, 65536, kvdgen.FP16)   # 2 KiB spans, 64k blocks
    pair = make_pair(g, g, seed=76)
    try:
        pair.peer.set(kvd.OPT_COALESCE, 0)
        rng = np.random.default_rng(0)
        n = 60000
        stop = threading.Event()
        polls = []
        target = [None]

        def poller():
            while not stop.is_set():
                rid = target[0]
                if rid is None:
                    continue
                t0 = time.perf_counter_ns()
                try:
                    done = pair.peer.poll(rid)
                except kvd.KvdError:
                    done = True
                dt = time.perf_counter_ns() - t0
                if not done:
                    polls.append(dt)

        th = threading.Thread(target=poller)
        th.start()
        pulls = []
        side = torch.cuda.Stream()
        try:
            for it in range(6):
                # `target` stays in flight behind a ~20 ms sleep on its stream
                rid = next_request_id()
                with torch.cuda.stream(side):
                    torch.cuda._sleep(40_000_000)
                pair.peer.pull(rid, [65535 - it], [65535 - it], side)
                target[0] = rid
                for _ in range(3):
                    s = rng.choice(65000, n, replace=False).astype(np.int32)
                    d = rng.choice(65000, n, replace=False).astype(np.int32)
                    r = next_request_id()
                    t0 = time.perf_counter_ns()
                    pair.peer.pull(r, s, d)
                    pulls.append(time.perf_counter_ns() - t0)
                    pair.peer.wait(r)
                target[0] = None
                side.synchronize()
                try:
                    pair.peer.wait(rid)
                except kvd.KvdError:
                    pass                                   # the poller retired it
        finally:
            stop.set()
            th.join()
        pull_med = float(np.median(pulls))
        assert len(polls) > 100, len(polls)
        p90 = float(np.percentile(polls, 90))
        print(f"kvd_pull median {pull_med / 1e3:.1f} us; poll p50 "
              f"{np.median(polls) / 1e3:.2f} us p90 {p90 / 1e3:.2f} us over {len(polls)} polls")
        assert p90 < 0.25 * pull_med, (p90, pull_med)
    finally:
        pair.close()


def test_batch_slot_reuse_while_batch_runs():
    """a TMA batch's counters belong to its descriptor buffer, not
    to request 0's completion slot.  Request 0 completes first; its id (hence
    its slot) is reused by a pull on a second stream while the batch is still
    moving its big requests; both stay bit-exact."""
    from paper_2501_14743_b200 import kvd
    g = kvdgen.CacheGeom(8, 8, 128, 16, 2048, kvdgen.BF16)    # 32 KiB spans
    pair = make_pair(g, g, seed=77)
    try:
        pair.peer.set(kvd.OPT_VARIANT, kvd.VARIANT_TMA)
        tables = kvdgen.disjoint_fragmented_tables([1, 600, 600, 600, 40], 2048, 2048, seed=11)
        ids = [next_request_id() for _ in range(4)]
        pair.peer.pull_batch(ids, tables[:4])
        while not pair.peer.poll(ids[0]):
            pass
        still = [i for i in ids[1:] if not pair.peer.poll(i)]
        other = torch.cuda.Stream()
        s, d = tables[4]
        pair.peer.pull(ids[0], s, d, other)     # same id -> request 0's slot
        pair.peer.wait(ids[0])
        for i in still:
            pair.peer.wait(i)
        print(f"{len(still)} batch requests were still in flight at the reuse")
        exp = pair.dst_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
        # the batch buffer is reused by the next batch once its kernel ended
        ids2 = [next_request_id() for _ in range(2)]
        t2 = kvdgen.disjoint_fragmented_tables([50, 50], 2048, 2048, seed=12)
        pre = pair.download_dst()
        pair.peer.pull_batch(ids2, t2)
        for i in ids2:
            pair.peer.wait(i)
        exp = pre
        for s, d in t2:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("engine", [0, 8])
def test_threads_mix_pulls_batches_and_polls(engine):
    """Stress: four issuing threads (single pulls of mixed sizes -- with the
    resident engine on, the short ones are posted to it and the long ones
    launched -- and batched drains, on their own streams) while a fifth
    thread retires completions with kvd_poll_many; a few hundred requests,
    disjoint destinations, then the whole cache against the oracle."""
    g = kvdgen.CacheGeom(2, 2, 64, 16, 8192, kvdgen.FP16)   # 4 KiB spans, 16 KiB per block
    pair = make_pair(g, g, seed=75)
    try:
        if engine:
            pair.peer.set(kvd.OPT_ENGINE, engine)
        rng = np.random.default_rng(engine)
        sizes = [int(x) for x in rng.choice([1, 3, 8, 40, 200], 1600,
                                            p=[0.3, 0.3, 0.25, 0.1, 0.05])]
        while sum(sizes) > 6500:               # ~80 % of the pool (room for gaps)
            sizes.pop()
        tables = kvdgen.disjoint_fragmented_tables(sizes, 8192, 8192, seed=11)
        ids = [next_request_id() for _ in tables]
        issued, errors, lock = [], [], threading.Lock()

        def issuer(w):
            try:
                stream = torch.cuda.Stream()
                k = w
                while k < len(tables):
                    batch = k % 7 == 3 and k + 4 < len(tables)   # a batch of this thread's next 2
                    ks = [k, k + 4] if batch else [k]
                    while True:
                        try:
                            if batch:
                                pair.peer.pull_batch([ids[q] for q in ks],
                                                     [tables[q] for q in ks], stream)
                            else:
                                pair.peer.pull(ids[k], *tables[k], stream)
                            break
                        except kvd.KvdError as e:                # all slots in flight
                            if e.status != kvd.EBUSY:
                                raise
                            time.sleep(1e-4)
                    k += 8 if batch else 4
                    with lock:
                        issued.extend(ids[q] for q in ks)
            except Exception as e:   # pragma: no cover - reported below
                errors.append(e)

        done = set()

        def poller():
            try:
                while len(done) < len(tables) and not errors:
                    with lock:
                        pending = [r for r in issued if r not in done]
                    if pending:
                        done.update(pair.peer.poll_many(pending))
            except Exception as e:   # pragma: no cover
                errors.append(e)

        threads = [threading.Thread(target=issuer, args=(w,)) for w in range(4)]
        threads.append(threading.Thread(target=poller))
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errors, errors
        assert done == set(ids)
        exp = pair.dst_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()
