"""Row-slab sharding of one atlas across ranks.

Texel queries are independent, so the atlas is split into contiguous row
ranges balanced by valid-texel count (skyline-packed atlases fill from row 0,
so equal row slabs would be unbalanced, pack.cpp:25-48). Each rank bakes its
rows - the library rasterises and transfers `radius` halo rows on each side
itself, so the dilated slab is exact without any exchange - and one
all-gather of the RGB8 slabs (padded to the largest slab) assembles the
row-major atlas on every rank. The BVH is built per rank (replicated).

`PeerAtlas` is the fused alternative: every rank exports its full-atlas
buffer over CUDA IPC, opens its peers', and the bake's dilation kernel stores
each output row straight into all of them (`mf_bake_normal_map_dev_publish`),
so the gather rides on the producing kernel's stores over NVLink instead of
a separate NCCL collective; one host barrier then marks every atlas complete.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np


def balanced_row_ranges(row_counts: Sequence[int], k: int) -> List[Tuple[int, int]]:
    """Split rows [0, R) into k contiguous non-empty ranges whose valid-texel
    counts are as equal as the prefix sums allow (ties go to equal rows)."""
    counts = np.asarray(row_counts, dtype=np.int64)
    rows = counts.size
    if k < 1 or k > rows:
        raise ValueError(f"cannot split {rows} rows into {k} ranges")
    weight = counts + 1  # every row costs something (rasterisation, dilation)
    csum = np.concatenate([[0], np.cumsum(weight)])
    total = csum[-1]
    cuts = [0]
    for r in range(1, k):
        target = total * r / k
        c = int(np.searchsorted(csum, target, side="left"))
        c = min(max(c, cuts[-1] + 1), rows - (k - r))
        cuts.append(c)
    cuts.append(rows)
    return [(cuts[i], cuts[i + 1]) for i in range(k)]


def pad_rows(slab, rows: int):
    """Pad a (r, W, C) slab to `rows` rows with zeros (numpy or torch)."""
    r = slab.shape[0]
    if r == rows:
        return slab
    try:
        import torch
        if isinstance(slab, torch.Tensor):
            out = torch.zeros((rows,) + tuple(slab.shape[1:]), dtype=slab.dtype, device=slab.device)
            out[:r] = slab
            return out
    except ImportError:  # pragma: no cover
        pass
    out = np.zeros((rows,) + slab.shape[1:], dtype=slab.dtype)
    out[:r] = slab
    return out


def assemble(gathered: Sequence, ranges: Sequence[Tuple[int, int]]):
    """Concatenate the (padded) per-rank slabs back into the full atlas."""
    parts = [g[: e - b] for g, (b, e) in zip(gathered, ranges)]
    try:
        import torch
        if isinstance(parts[0], torch.Tensor):
            return torch.cat(parts, 0)
    except ImportError:  # pragma: no cover
        pass
    return np.concatenate(parts, 0)


def sharded_bake(bake_rows: Callable[[int, int], object], ranges: Sequence[Tuple[int, int]], rank: int,
                 group=None):
    """Bake this rank's rows with `bake_rows(b, e)` (returns a (e-b, W, 3)
    uint8 slab, numpy on CPU/gloo or a CUDA tensor on NCCL) and all-gather
    the slabs into the full atlas on every rank."""
    import torch
    import torch.distributed as dist

    b, e = ranges[rank]
    slab = bake_rows(b, e)
    rows_max = max(hi - lo for lo, hi in ranges)
    as_tensor = torch.as_tensor(pad_rows(slab, rows_max))
    gathered = [torch.empty_like(as_tensor) for _ in ranges]
    dist.all_gather(gathered, as_tensor.contiguous(), group=group)
    return assemble(gathered, ranges)


class PeerAtlas:
    """Full-atlas buffers shared by all ranks of a node through CUDA IPC.

    `atlas` is this rank's (res, res, 3) uint8 CUDA tensor; `dst` holds the
    device pointers of every rank's atlas as seen from this process (own
    first), ready for mf_bake_normal_map_dev_publish."""

    def __init__(self, ctx, res: int, group=None):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import capi

        self.ctx = ctx
        self.atlas = torch.zeros((res, res, 3), dtype=torch.uint8, device="cuda")
        handle = (ctypes.c_uint8 * 64)()
        offset = ctypes.c_uint64(0)
        capi.check(ctx.lib.mf_ipc_export(ctypes.c_void_p(self.atlas.data_ptr()), handle, ctypes.byref(offset)))
        mine = (bytes(handle), int(offset.value))
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        every = [None] * world
        dist.all_gather_object(every, mine, group=group)
        self.opened = []
        ptrs = [self.atlas.data_ptr()]
        for r in range(world):
            if r == rank:
                continue
            h = (ctypes.c_uint8 * 64).from_buffer_copy(every[r][0])
            p = ctypes.c_void_p()
            capi.check(ctx.lib.mf_ipc_open(ctx.h, h, ctypes.c_uint64(every[r][1]), ctypes.byref(p)))
            self.opened.append(p.value)
            ptrs.append(p.value)
        self.dst = (ctypes.c_void_p * len(ptrs))(*ptrs)
        self.n = len(ptrs)

    def close(self):
        import ctypes
        for p in self.opened:
            self.ctx.lib.mf_ipc_close(self.ctx.h, ctypes.c_void_p(p))
        self.opened = []
