"""Shared helpers of the GPU parity tests (test infrastructure).

Caches are filled with seeded inputs from kvdgen; the expected result always
comes from the CPU oracle (oracle/kvd_oracle.c) run on host copies of those
inputs -- never from the CUDA path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np
import torch

import kvdgen
from oracle import oracle
from paper_2501_14743_b200 import kvd
from paper_2501_14743_b200.torch_cache import PagedCache, Peer


def cache_for(geom: kvdgen.CacheGeom, device: int, single_allocation=False,
              memory="torch", mem_kind=kvd.MEM_AUTO) -> PagedCache:
    return PagedCache(geom.num_layers, geom.num_kv_heads, geom.head_dim, geom.block_size,
                      geom.num_blocks, geom.dtype, geom.stride, device,
                      single_allocation=single_allocation, memory=memory, mem_kind=mem_kind)


def oracle_layer_bytes(geom: kvdgen.CacheGeom) -> int:
    stride = geom.stride if any(geom.stride) else oracle.default_strides(
        geom.num_blocks, geom.block_size, geom.num_kv_heads, geom.head_dim)
    return oracle.layer_nbytes(stride, geom.num_blocks, geom.block_size, geom.num_kv_heads,
                               geom.head_dim, geom.elem_bytes)


@dataclass
class Pair:
    sg: kvdgen.CacheGeom
    dg: kvdgen.CacheGeom
    src: PagedCache
    dst: PagedCache
    peer: Peer
    src_host: List[np.ndarray]
    dst_host: List[np.ndarray]     # pre-state of the destination

    def upload_dst(self, host: List[np.ndarray]):
        for l, h in enumerate(host):
            self.dst.layers[l].copy_(torch.from_numpy(h))
        torch.cuda.synchronize(self.dst.device)

    def download_dst(self) -> List[np.ndarray]:
        torch.cuda.synchronize(self.dst.device)
        return [t.cpu().numpy() for t in self.dst.layers]

    def expected(self, src_ids, dst_ids, pre=None) -> List[np.ndarray]:
        exp = [d.copy() for d in (pre if pre is not None else self.dst_host)]
        rc = oracle.pull(self.src_host, self.sg.stride, self.sg.num_blocks, exp,
                         self.dg.stride, self.dg.num_blocks, self.sg.num_kv_heads,
                         self.sg.head_dim, self.sg.block_size, self.sg.elem_bytes,
                         np.asarray(src_ids, np.int32), np.asarray(dst_ids, np.int32))
        assert rc == oracle.OK
        return exp

    def close(self):
        self.peer.close()
        self.dst.close()
        self.src.close()


def make_pair(sg: kvdgen.CacheGeom, dg: kvdgen.CacheGeom, seed: int, src_dev=0, dst_dev=0,
              single_allocation=False, src_memory="torch", dst_memory="torch") -> Pair:
    src = cache_for(sg, src_dev, single_allocation, src_memory)
    dst = cache_for(dg, dst_dev, single_allocation, dst_memory)
    assert src.layer_bytes == oracle_layer_bytes(sg)
    assert dst.layer_bytes == oracle_layer_bytes(dg)
    src_host = [kvdgen.random_bytes(src.layer_bytes, seed * 7919 + l) for l in range(sg.num_layers)]
    dst_host = [kvdgen.random_bytes(dst.layer_bytes, seed * 7919 + 100003 + l)
                for l in range(dg.num_layers)]
    for l in range(sg.num_layers):
        src.layers[l].copy_(torch.from_numpy(src_host[l]))
        dst.layers[l].copy_(torch.from_numpy(dst_host[l]))
    torch.cuda.synchronize()
    peer = dst.open_peer(src.export())
    return Pair(sg, dg, src, dst, peer, src_host, dst_host)


def assert_layers_equal(got: List[np.ndarray], exp: List[np.ndarray]):
    for l, (g, e) in enumerate(zip(got, exp)):
        if not np.array_equal(g, e):
            bad = np.flatnonzero(g != e)
            raise AssertionError(f"layer {l}: {bad.size} bytes differ, first at byte {bad[0]} "
                                 f"(got {g[bad[0]]}, want {e[bad[0]]})")


_req = [1000]


def next_request_id() -> int:
    _req[0] += 1
    return _req[0]


def pull_and_wait(pair: Pair, src_ids, dst_ids, request_id=None, timeout_us=30_000_000) -> dict:
    rid = next_request_id() if request_id is None else request_id
    pair.peer.pull(rid, src_ids, dst_ids)
    pair.peer.wait(rid, timeout_us)
    return pair.peer.info()
