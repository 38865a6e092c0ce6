"""GPU: the row-sharded bake whose dilation kernel publishes each output row
into every rank's atlas over CUDA IPC peer memory (
mf_bake_normal_map_dev_publish). Two processes on the one available GPU
(gloo for the host rendezvous and barrier) each bake half of the atlas's rows
into both atlases; both must equal a single-process full bake byte for byte."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, out_dir):
    import ctypes

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_26137_b200 import capi, fixtures as fx, sharding

    pair = fx.bake_pair(n_dense=48, n_low=8, res=256, name="publish")
    ctx = capi.Context(0, torch.cuda.current_stream().cuda_stream)
    lo, hi = capi.DeviceMesh(ctx, pair.lowpoly), capi.DeviceMesh(ctx, pair.dense)
    counts = np.zeros(pair.res, np.int64)
    capi.check(ctx.lib.mf_coverage_rows(ctx.h, lo.h, pair.res, ctypes.c_void_p(counts.ctypes.data)))
    ranges = sharding.balanced_row_ranges(counts, world)
    peer = sharding.PeerAtlas(ctx, pair.res)
    b, e = ranges[rank]
    for _ in range(3):  # eager, capture, replay
        capi.check(ctx.lib.mf_bake_normal_map_dev_publish(ctx.h, lo.h, hi.h, pair.res, pair.bbox_diagonal,
                                                          pair.max_distance_fraction, 4, b, e, peer.dst, peer.n,
                                                          None))
        torch.cuda.synchronize()
        dist.barrier()
    np.save(os.path.join(out_dir, f"atlas{rank}.npy"), peer.atlas.cpu().numpy())
    if rank == 0:
        full = torch.empty((pair.res, pair.res, 3), dtype=torch.uint8, device="cuda")
        capi.check(ctx.lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, pair.res, pair.bbox_diagonal,
                                                  pair.max_distance_fraction, 4, 0, pair.res, full.data_ptr(), None))
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, "full.npy"), full.cpu().numpy())
    dist.barrier()
    peer.close()
    dist.destroy_process_group()


def test_publish_gather_two_ranks_one_gpu(gpu_ctx, tmp_path):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    full = np.load(tmp_path / "full.npy")
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"atlas{r}.npy"), full), f"rank {r} atlas differs"
