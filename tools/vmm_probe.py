"""Probe the box for the f3 handle kinds: fabric handles (multi-node NVLink /
IMEX) and POSIX-fd VMM handles, plus whether a sibling process can fetch an
exported fd with pidfd_getfd (the fd-passing route that needs no socket).

    python tools/vmm_probe.py > gpurun_out/vmm_probe.json
"""
import ctypes
import json
import multiprocessing as mp
import os

from cuda.bindings import driver as cu


def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    rest = r[1:] if isinstance(r, tuple) else ()
    return err, (rest[0] if len(rest) == 1 else rest)


def prop(handle_type, dev=0):
    p = cu.CUmemAllocationProp()
    p.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    p.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    p.location.id = dev
    p.requestedHandleTypes = handle_type
    return p


def child(pid, fd, q):
    libc = ctypes.CDLL(None, use_errno=True)
    SYS_pidfd_open, SYS_pidfd_getfd = 434, 438
    pidfd = libc.syscall(SYS_pidfd_open, pid, 0)
    if pidfd < 0:
        q.put({"pidfd_open": os.strerror(ctypes.get_errno())})
        return
    nfd = libc.syscall(SYS_pidfd_getfd, pidfd, fd, 0)
    out = {"pidfd_getfd": "ok" if nfd >= 0 else os.strerror(ctypes.get_errno())}
    if nfd >= 0:
        cu.cuInit(0)
        err, dev = chk(cu.cuDeviceGet(0))
        err, ctx = chk(cu.cuDevicePrimaryCtxRetain(dev))
        cu.cuCtxSetCurrent(ctx)
        err, h = chk(cu.cuMemImportFromShareableHandle(
            nfd, cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR))
        out["import_posix_fd"] = str(err)
    q.put(out)


def main():
    res = {}
    try:
        res["ptrace_scope"] = open("/proc/sys/kernel/yama/ptrace_scope").read().strip()
    except OSError as e:
        res["ptrace_scope"] = str(e)
    cu.cuInit(0)
    err, dev = chk(cu.cuDeviceGet(0))
    for name in ("CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_GPU_DIRECT_RDMA_WITH_CUDA_VMM_SUPPORTED"):
        err, v = chk(cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, name), dev))
        res[name] = v if err == cu.CUresult.CUDA_SUCCESS else str(err)
    err, ctx = chk(cu.cuDevicePrimaryCtxRetain(dev))
    cu.cuCtxSetCurrent(ctx)
    HT = cu.CUmemAllocationHandleType
    err, gran = chk(cu.cuMemGetAllocationGranularity(
        prop(HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
        cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
    res["granularity"] = gran
    # fabric
    err, h = chk(cu.cuMemCreate(gran, prop(HT.CU_MEM_HANDLE_TYPE_FABRIC), 0))
    res["create_fabric"] = str(err)
    if err == cu.CUresult.CUDA_SUCCESS:
        err2, fh = chk(cu.cuMemExportToShareableHandle(h, HT.CU_MEM_HANDLE_TYPE_FABRIC, 0))
        res["export_fabric"] = str(err2)
        cu.cuMemRelease(h)
    # posix fd
    err, h = chk(cu.cuMemCreate(gran, prop(HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), 0))
    res["create_posix_fd"] = str(err)
    if err == cu.CUresult.CUDA_SUCCESS:
        err2, fd = chk(cu.cuMemExportToShareableHandle(
            h, HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0))
        res["export_posix_fd"] = str(err2)
        if err2 == cu.CUresult.CUDA_SUCCESS:
            ctxm = mp.get_context("spawn")
            q = ctxm.Queue()
            p = ctxm.Process(target=child, args=(os.getpid(), int(fd), q))
            p.start()
            res["child"] = q.get(timeout=120)
            p.join()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
