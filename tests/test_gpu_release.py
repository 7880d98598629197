"""Complete() toward the prefill side: every completed pull
posts its request id into the exporter's release mailbox; the exporter's
kvd_poll_released returns each id exactly once, after its bytes landed."""
import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, make_pair, next_request_id, pull_and_wait
from paper_2501_14743_b200 import kvd

pytestmark = pytest.mark.gpu

G = kvdgen.CacheGeom(2, 2, 64, 16, 256, kvdgen.FP16)


def _exercise(pair):
    ids = []
    for k in range(3):                                    # single pulls
        s, d = kvdgen.random_table(10 + k, 256, 256, seed=k)
        rid = next_request_id()
        pair.peer.pull(rid, s, d)
        pair.peer.wait(rid)
        ids.append(rid)
    rid = next_request_id()                               # n = 0
    pair.peer.pull(rid, [], [])
    pair.peer.wait(rid)
    ids.append(rid)
    tables = kvdgen.disjoint_fragmented_tables([7, 0, 12], 256, 256, seed=9)
    bids = [next_request_id() for _ in tables]            # batched drain
    pair.peer.pull_batch(bids, tables)
    for b in bids:
        pair.peer.wait(b)
    return ids + bids


def test_release_mailbox_loopback():
    pair = make_pair(G, G, seed=60)
    try:
        assert pair.src.poll_released() == []
        ids = _exercise(pair)
        torch.cuda.synchronize()
        got = pair.src.poll_released()
        assert sorted(got) == sorted(ids) and len(got) == len(set(got))
        assert pair.src.poll_released() == []             # each id once
        more = _exercise(pair)
        got = []
        for _ in range(100):
            got += pair.src.poll_released(cap=3)          # small cap: resumes in order
            if len(got) == len(more):
                break
        assert sorted(got) == sorted(more)
    finally:
        pair.close()


def test_release_after_bytes_landed():
    """The release id is posted only after the request's last read: once an
    id is observed, the destination already holds every pulled byte."""
    pair = make_pair(G, G, seed=61)
    span = pair.src.span_bytes
    src_view = [torch.from_numpy(h).view(2, 256, span) for h in pair.src_host]
    try:
        for it in range(200):
            s, d = kvdgen.random_table(int(np.random.default_rng(it).integers(1, 40)), 256, 256,
                                       seed=100 + it)
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            got = []
            while rid not in got:
                got += pair.src.poll_released()
            for l in range(G.num_layers):
                now = pair.dst.layers[l].view(2, 256, span)[:, torch.from_numpy(d).long().cuda()].cpu()
                assert torch.equal(now, src_view[l][:, torch.from_numpy(s).long()])
            pair.peer.wait(rid)
    finally:
        pair.close()


def test_push_does_not_post_releases():
    pair = make_pair(G, G, seed=62)
    try:
        rev = pair.src.open_peer(pair.dst.export())
        rid = next_request_id()
        rev.push(rid, [1, 2], [3, 4])
        rev.wait(rid)
        torch.cuda.synchronize()
        assert pair.dst.poll_released() == []
        rev.close()
    finally:
        pair.close()


@pytest.mark.gpu2
def test_release_mailbox_two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    pair = make_pair(G, G, seed=63, src_dev=0, dst_dev=1)
    try:
        ids = _exercise(pair)
        torch.cuda.synchronize(1)
        got = pair.src.poll_released()
        assert sorted(got) == sorted(ids)
    finally:
        pair.close()


def test_poll_released_does_not_wait_for_exporter_work():
    """The exporter polls while its own GPU is busy (prefill kernels queued on
    the default stream): the poll must not serialise behind that work."""
    import time
    pair = make_pair(G, G, seed=64)
    try:
        s, d = kvdgen.random_table(20, 256, 256, seed=5)
        rid = next_request_id()
        pair.peer.pull(rid, s, d)
        pair.peer.wait(rid)
        torch.cuda._sleep(1_500_000_000)          # ~0.75 s of "prefill" on the default stream
        t0 = time.perf_counter()
        got = pair.src.poll_released()
        dt = time.perf_counter() - t0
        torch.cuda.synchronize()
        assert got == [rid]
        assert dt < 0.3, f"poll_released waited {dt:.3f} s behind the default stream"
    finally:
        pair.close()


def test_release_rings_per_importer():
    """The mailbox is host memory shared by the exporter and its importers;
    each open peer owns one single-producer ring (64 at a time).  Two
    importers' releases both reach the exporter; a closed importer's ring is
    reused by the next one, which continues its positions; a 65th importer
    is refused with KVD_EBUSY."""
    from gpu_helpers import cache_for
    pair = make_pair(G, G, seed=65)
    extra = []
    try:
        other = cache_for(G, 0)
        extra.append(other)
        p2 = other.open_peer(pair.src.export())
        ids1, ids2 = [], []
        for k in range(5):
            s, d = kvdgen.random_table(9, 256, 256, seed=40 + k)
            r1, r2 = next_request_id(), next_request_id()
            pair.peer.pull(r1, s, d)
            p2.pull(r2, s, d)
            ids1.append(r1)
            ids2.append(r2)
        for r in ids1:
            pair.peer.wait(r)
        for r in ids2:
            p2.wait(r)
        assert sorted(pair.src.poll_released()) == sorted(ids1 + ids2)
        p2.close()
        p3 = other.open_peer(pair.src.export())           # takes the freed ring
        r3 = next_request_id()
        p3.pull(r3, [5], [6])
        p3.wait(r3)
        assert pair.src.poll_released() == [r3]
        peers = [p3]
        with pytest.raises(kvd.KvdError) as ei:
            for _ in range(70):
                peers.append(other.open_peer(pair.src.export()))
        assert ei.value.status == kvd.EBUSY
        assert len(peers) == 63                           # + pair.peer = 64 rings
        for p in peers:
            p.close()
    finally:
        pair.close()
        for c in extra:
            c.close()
