"""Multi-process (gloo, world size 2, CPU) checks of the N > 1 path: RHS sharding with the
operator replicated and no data-path collective; max-over-ranks timing.  The per-rank
apply is the oracle's (a CPU stand-in for xc_apply): columns are independent, so the
concatenated shards must equal the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2004_11610_b200.shard import column_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import oracle as O
    from paper_2004_11610_b200 import inputs as I
    from paper_2004_11610_b200.shard import column_shard, max_over_ranks, sum_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, B = 256, 10
    kind = O.Kind(O.KIND_JACOBI, 0.5, -0.3)
    x, _, _ = O.gauss_rule(kind, N)                 # replicated operator
    op = O.compress(O.make_plan(kind, N, 1e-12), x)
    X = I.rhs(N, B, 21)
    sl = column_shard(B, rank, world)
    Y = O.apply_output_axis(op, X[:, sl])           # this rank's columns only
    np.save(os.path.join(out_dir, f"y{rank}.npy"), Y)
    mx = max_over_ranks(10.0 + rank)
    tot = sum_over_ranks(sl.stop - sl.start)
    np.save(os.path.join(out_dir, f"m{rank}.npy"), np.array([mx, tot]))
    dist.barrier()
    dist.destroy_process_group()


def test_column_shard_partition():
    for B in (1, 7, 64, 4096):
        for G in (1, 2, 3, 8):
            cols = np.concatenate([np.arange(B)[column_shard(B, g, G)] for g in range(G)])
            assert np.array_equal(cols, np.arange(B))
    with pytest.raises(ValueError):
        column_shard(8, 2, 2)


def test_two_rank_gloo_shards_equal_single_process(tmp_path):
    import oracle as O
    from paper_2004_11610_b200 import inputs as I
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    N, B = 256, 10
    kind = O.Kind(O.KIND_JACOBI, 0.5, -0.3)
    x, _, _ = O.gauss_rule(kind, N)
    op = O.compress(O.make_plan(kind, N, 1e-12), x)
    Yfull = O.apply_output_axis(op, I.rhs(N, B, 21))
    Ycat = np.concatenate([np.load(tmp_path / f"y{r}.npy") for r in range(2)], axis=1)
    # the GPU path is bit-identical per column (tests/test_gpu_parity.py); the CPU stand-in's
    # library FFT/sparse kernels may block differently with the batch width
    assert np.abs(Ycat - Yfull).max() <= 1e-14 * np.abs(Yfull).max()
    for r in range(2):
        mx, tot = np.load(tmp_path / f"m{r}.npy")
        assert mx == 11.0 and tot == B


def _ag_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2004_11610_b200 import xc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 13 + 0  # bytes per rank (odd on purpose)
    send = torch.arange(n, dtype=torch.uint8) + 100 * rank
    recv = torch.empty(n * world, dtype=torch.uint8)
    xc.nccl_allgather()(send, recv)   # the binding's exchange: rank-major all-gather
    np.save(os.path.join(out_dir, f"ag{rank}.npy"), recv.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_exchange_layout(tmp_path):
    """The distributed precompute's exchange contract (include/xc.h, xc_exchange_t): recv holds
    rank r's send at offset r * bytes_per_rank on every rank."""
    port = _free_port()
    mp.spawn(_ag_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    want = np.concatenate([np.arange(13, dtype=np.uint8) + 100 * r for r in range(2)])
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"ag{r}.npy"), want)
