#!/usr/bin/env python
"""Probe (one GPU): can this box give the extraction epilogue an NVLS multicast address?

Checks CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, a 1-device multicast object through the
driver API (cuMulticastCreate / AddDevice / BindMem / Map), and torch's symmetric memory
(symm_mem.rendezvous -> multicast_ptr) on a 1-rank NCCL group.  Prints one JSON line."""
import json
import os

import torch


def driver_probe():
    import cuda.bindings.driver as d
    out = {}
    (err,) = d.cuInit(0)
    err, dev = d.cuDeviceGet(0)
    err, v = d.cuDeviceGetAttribute(
        d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    out["attr_multicast_supported"] = int(v)
    err, ctx = d.cuDevicePrimaryCtxRetain(dev)
    d.cuCtxSetCurrent(ctx)
    for attr in ("CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
        a = getattr(d.CUdevice_attribute, attr, None)
        if a is not None:
            out[attr] = int(d.cuDeviceGetAttribute(a, dev)[1])
    H = d.CUmemAllocationHandleType
    for name, ht in (("none", 0), ("posix_fd", H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                     ("fabric", getattr(H, "CU_MEM_HANDLE_TYPE_FABRIC", None))):
        if ht is None:
            continue
        r = {}
        prop = d.CUmulticastObjectProp()
        prop.numDevices = 1
        prop.size = 2 << 20
        prop.handleTypes = ht
        prop.flags = 0
        err, gran = d.cuMulticastGetGranularity(
            prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        r["granularity"] = [str(err), int(gran) if err == d.CUresult.CUDA_SUCCESS else None]
        if err == d.CUresult.CUDA_SUCCESS:
            prop.size = max(int(gran), 2 << 20)
            err, mc = d.cuMulticastCreate(prop)
            r["create"] = str(err)
            if err == d.CUresult.CUDA_SUCCESS:
                (err,) = d.cuMulticastAddDevice(mc, dev)
                r["add_device"] = str(err)
        out[name] = r
    return out


def symm_probe():
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    out = {}
    try:
        t = symm_mem.empty(1 << 22, dtype=torch.uint8, device=dev)
        h = symm_mem.rendezvous(t, dist.group.WORLD)
        out["world"] = h.world_size
        from torch._C._distributed_c10d import _SymmetricMemory
        out["has_multicast_support"] = bool(_SymmetricMemory.has_multicast_support(
            torch._C._autograd.DeviceType.CUDA, 0)) if hasattr(torch._C, "_autograd") else None
        out["multicast_ptr"] = int(h.multicast_ptr)
        out["buffer_ptr0"] = int(h.buffer_ptrs[0])
    except Exception as e:  # noqa: BLE001
        out["error"] = repr(e)[:300]
    dist.destroy_process_group()
    return out


if __name__ == "__main__":
    res = {}
    try:
        res["driver"] = driver_probe()
    except Exception as e:  # noqa: BLE001
        res["driver_error"] = repr(e)[:300]
    try:
        res["symm_mem"] = symm_probe()
    except Exception as e:  # noqa: BLE001
        res["symm_error"] = repr(e)[:300]
    print(json.dumps(res))
