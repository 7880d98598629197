"""Paged KV caches as torch device memory, registered with libkvd.

torch is only the allocator and stream provider here: a ``PagedCache`` owns
one uint8 tensor per layer (vLLM keeps one tensor per layer) -- or one
tensor sliced into layers -- sized by the library's own geometry
(kvd_layout_geometry), and registers the layer bases with
kvd_register_cache.  Every byte of a pull is moved by libkvd's kernel.
With ``memory="vmm"`` the cache lives in one kvd_mem_alloc allocation (CUDA
VMM, exported as a POSIX fd or fabric handle -- §8 f3 groundwork) that torch
only views through ``__cuda_array_interface__``.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from . import kvd


class _DeviceBytes:
    """A raw device range as a CUDA-array-interface object (no ownership)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class PagedCache:
    def __init__(self, num_layers: int, num_kv_heads: int, head_dim: int, block_size: int,
                 num_blocks: int, dtype: int = kvd.FP16, stride: Sequence[int] = (0,) * 5,
                 device: int = 0, single_allocation: bool = False, pad_bytes: int = 0,
                 memory: str = "torch", mem_kind: int = kvd.MEM_AUTO):
        self.layout = kvd.make_layout(num_layers, num_kv_heads, head_dim, block_size, num_blocks,
                                      dtype, stride)
        self.geom = kvd.kvd_layout_geometry(self.layout)
        self.device = int(device)
        self.layer_bytes = int(self.geom.layer_bytes)
        # round each layer to 512 B so every base stays 32 B aligned
        self.layer_pitch = (self.layer_bytes + pad_bytes + 511) // 512 * 512
        dev = torch.device("cuda", self.device)
        self._vmm_ptr = None
        self.mem_kind = None
        if memory == "vmm":
            ptr, _, self.mem_kind = kvd.kvd_mem_alloc(self.device, self.layer_pitch * num_layers,
                                                      mem_kind)
            self._vmm_ptr = ptr
            with torch.cuda.device(self.device):
                self._storage = torch.as_tensor(
                    _DeviceBytes(ptr, self.layer_pitch * num_layers), device=dev)
            self.layers = [
                self._storage[l * self.layer_pitch:l * self.layer_pitch + self.layer_bytes]
                for l in range(num_layers)]
        elif memory != "torch":
            raise ValueError(f"memory must be 'torch' or 'vmm', not {memory!r}")
        elif single_allocation:
            self._storage = torch.empty(self.layer_pitch * num_layers, dtype=torch.uint8,
                                        device=dev)
            self.layers: List[torch.Tensor] = [
                self._storage[l * self.layer_pitch:l * self.layer_pitch + self.layer_bytes]
                for l in range(num_layers)]
        else:
            self._storage = None
            self.layers = [torch.empty(self.layer_bytes, dtype=torch.uint8, device=dev)
                           for _ in range(num_layers)]
        self.handle: Optional[int] = kvd.kvd_register_cache(
            self.device, self.layout, [t.data_ptr() for t in self.layers])

    @property
    def num_blocks(self) -> int:
        return self.layout.num_blocks

    @property
    def span_bytes(self) -> int:
        return int(self.geom.span_bytes)

    def export(self) -> bytes:
        return kvd.kvd_export_handle(self.handle)

    def open_peer(self, blob: bytes) -> "Peer":
        return Peer(self, kvd.kvd_open_peer(self.handle, blob))

    def poll_released(self, cap: int = 4096) -> list:
        """Exporter side of Complete(): ids of requests pulled from
        this cache that have completed since the last call."""
        return kvd.kvd_poll_released(self.handle, cap)

    def open_peer_heads(self, blob: bytes, head_offset: int) -> "Peer":
        """§8 f4: the blob's (fewer) heads land at heads [head_offset, ...)."""
        return Peer(self, kvd.kvd_open_peer_heads(self.handle, blob, head_offset))

    def close(self) -> None:
        """Unregister; a ``memory="vmm"`` cache also frees its memory (the
        layer tensors are invalid afterwards)."""
        if self.handle:
            kvd.kvd_unregister_cache(self.handle)
            self.handle = None
        if self._vmm_ptr:
            self.layers, self._storage = [], None
            kvd.kvd_mem_free(self._vmm_ptr)
            self._vmm_ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Peer:
    """Decode-side binding of a prefill cache (kvd_peer)."""

    def __init__(self, local: PagedCache, handle: int):
        self.local = local
        self.handle: Optional[int] = handle

    def set(self, option: int, value: int) -> "Peer":
        kvd.kvd_peer_set(self.handle, option, value)
        return self

    def pull(self, request_id: int, src_ids, dst_ids, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.local.device)
        kvd.kvd_pull(self.handle, request_id, src_ids, dst_ids, s.cuda_stream)

    def push(self, request_id: int, src_ids, dst_ids, stream: Optional[torch.cuda.Stream] = None):
        """§8 f2: local blocks -> the imported cache's blocks (stores over NVLink)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.local.device)
        kvd.kvd_push(self.handle, request_id, src_ids, dst_ids, s.cuda_stream)

    def pull_batch(self, request_ids, tables, stream: Optional[torch.cuda.Stream] = None):
        """§8 f1: several requests, one launch, per-request completion."""
        s = stream if stream is not None else torch.cuda.current_stream(self.local.device)
        kvd.kvd_pull_batch(self.handle, request_ids, tables, s.cuda_stream)

    def poll(self, request_id: int) -> bool:
        return kvd.kvd_poll_done(self.handle, request_id)

    def poll_many(self, request_ids) -> list:
        """Completed (and now retired) ids among `request_ids`, one C call."""
        return kvd.kvd_poll_many(self.handle, request_ids)

    def wait(self, request_id: int, timeout_us: int = 30_000_000) -> None:
        kvd.kvd_wait_done(self.handle, request_id, timeout_us)

    def audit(self) -> int:
        """Bounds-audit violations (KVD_OPT_AUDIT must be set)."""
        return kvd.kvd_peer_audit(self.handle)

    def kernel_time(self):
        """(kernel-only ms summed, launches) since the last call; needs OPT_TIMING."""
        return kvd.kvd_peer_kernel_time(self.handle)

    def device_time(self):
        """(ms, requests): in-kernel first-CTA-start -> last-CTA-done spans of the
        retired single pulls since the last call; needs OPT_TIMING."""
        return kvd.kvd_peer_device_time(self.handle)

    def calibrate(self, nbytes: int, ctas: int = 0, stages: int = 0, reps: int = 3) -> float:
        """Measured link ceiling (GB/s): discarded bulk reads of `nbytes` of the
        peer's source layers, no stores (kvd_peer_calibrate)."""
        return kvd.kvd_peer_calibrate(self.handle, nbytes, ctas, stages, reps)

    def spans(self) -> list:
        """[(request_id, start_ns, wait_ns, end_ns)] %globaltimer timelines of the
        timed single pulls retired since the last call; needs OPT_TIMING."""
        return kvd.kvd_peer_spans(self.handle)

    def stream_wait(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """With OPT_STREAMS >= 2: order `stream` after every transfer issued so far."""
        s = stream if stream is not None else torch.cuda.current_stream(self.local.device)
        kvd.kvd_stream_wait(self.handle, s.cuda_stream)

    def info(self) -> dict:
        return kvd.kvd_last_pull_info(self.handle).as_dict()

    def close(self) -> None:
        if self.handle:
            kvd.kvd_close_peer(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
