"""Cost of mapping device memory with the CUDA virtual-memory API on this
box (the lazily mapped population pool, engine.cu ensure_pool): per-granule
cuMemCreate / cuMemMap / cuMemSetAccess times for several granule sizes, with
and without a kernel keeping the GPU busy."""
import json
import time

import torch
from cuda.bindings import driver as d


def ck(r):
    if isinstance(r, tuple):
        if r[0] != d.CUresult.CUDA_SUCCESS:
            raise RuntimeError(r)
        return r[1] if len(r) == 2 else r[1:]
    if r != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(r)


def run(gran_mb, total_gb, busy):
    torch.cuda.init()
    prop = d.CUmemAllocationProp()
    prop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = 0
    acc = d.CUmemAccessDesc()
    acc.location = prop.location
    acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    g = gran_mb << 20
    n = int(total_gb * (1 << 30)) // g
    base = ck(d.cuMemAddressReserve(n * g, g, 0, 0))
    x = torch.empty(1 << 28, device="cuda") if busy else None
    t = {"create": 0.0, "map": 0.0, "access": 0.0}
    hs = []
    for k in range(n):
        if busy and k % 8 == 0:
            x.mul_(1.0000001)  # keep the GPU busy (queued work)
        t0 = time.perf_counter()
        h = ck(d.cuMemCreate(g, prop, 0))
        t1 = time.perf_counter()
        ck(d.cuMemMap(int(base) + k * g, g, 0, h, 0))
        t2 = time.perf_counter()
        ck(d.cuMemSetAccess(int(base) + k * g, g, [acc], 1))
        t3 = time.perf_counter()
        t["create"] += t1 - t0
        t["map"] += t2 - t1
        t["access"] += t3 - t2
        hs.append(h)
    torch.cuda.synchronize()
    # first touch
    t0 = time.perf_counter()
    ck(d.cuMemsetD8(int(base), 0, n * g))
    torch.cuda.synchronize()
    touch = time.perf_counter() - t0
    for k, h in enumerate(hs):
        ck(d.cuMemUnmap(int(base) + k * g, g))
        ck(d.cuMemRelease(h))
    ck(d.cuMemAddressFree(base, n * g))
    del x
    torch.cuda.empty_cache()
    gb = n * g / 1e9
    print(json.dumps({"granule_MiB": gran_mb, "GB": round(gb, 2), "busy": busy, "granules": n,
                      **{k + "_ms": round(v * 1e3, 1) for k, v in t.items()},
                      "ms_per_GB": round(sum(t.values()) * 1e3 / gb, 2),
                      "memset_GBs": round(gb / touch, 1)}), flush=True)


if __name__ == "__main__":
    for gran in (2, 64, 512, 2048):
        for busy in (False, True):
            run(gran, 32 if gran > 2 else 4, busy)
    t0 = time.perf_counter()
    y = torch.empty(int(32e9) // 4, device="cuda")
    torch.cuda.synchronize()
    print(json.dumps({"cudaMalloc_32GB_ms": round((time.perf_counter() - t0) * 1e3, 1)}))
