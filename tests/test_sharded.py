"""Row sharding over torch.distributed with world_size 2 on CPU (gloo).

The per-rank product is the CPU oracle on the rank's slab (test infrastructure); the plumbing
under test — slab bounds, x broadcast, ordered y gather, uneven slabs — is the same
RowShardedSpmv the GPU bench uses over NCCL.  Slab encodings must equal the global encoding
sliced, and the gathered y must equal the single-process y bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, R, C, d, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2511_13061_b200.sharded import RowShardedSpmv, slab_bounds

        r0, r1 = slab_bounds(R, world, rank)
        A = O.gen_dense(R, C, d, 7)[r0:r1]
        m = O.encode_dense(A)

        def local(x, y):
            xh = x.view(torch.int16).numpy().view(np.uint16)
            y.view(torch.int16).copy_(torch.from_numpy(O.reference_spmv(m, xh).view(np.int16)))

        sh = RowShardedSpmv(R, C, local)
        x = torch.zeros(C, dtype=torch.float16)
        if rank == 0:
            x.view(torch.int16).copy_(torch.from_numpy(O.gen_vector(C, 8).view(np.int16)))
        y = sh(x)
        if rank == 0:
            np.save(out_path, y.view(torch.int16).numpy().view(np.uint16))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("R,C,d", [(64, 300, 0.5), (37, 1000, 0.3)])  # even and uneven slabs
def test_row_sharded_spmv_gloo_world2(tmp_path, R, C, d):
    from oracle import oracle as O

    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(2, _free_port(), R, C, d, out), nprocs=2, join=True)
    y = np.load(out)
    A = O.gen_dense(R, C, d, 7)
    y_ref = O.reference_spmv(O.encode_dense(A), O.gen_vector(C, 8))
    assert np.array_equal(y, y_ref)


def test_slab_bounds_cover_rows():
    from paper_2511_13061_b200.sharded import slab_bounds

    for R, N in ((131072, 8), (36864, 4), (37, 2), (5, 8)):
        b = [slab_bounds(R, N, g) for g in range(N)]
        assert b[0][0] == 0 and b[-1][1] == R
        assert all(b[i][1] == b[i + 1][0] for i in range(N - 1))
        assert max(y - x for x, y in b) - min(y - x for x, y in b) <= 1


@pytest.mark.gpu
def test_nccl_sharded_spmv_single_rank(cuda):
    # macko_sharded_spmv over a real (one-rank) NCCL communicator: broadcast + slab SpMV +
    # in-place all-gather; y equals the plain SpMV.  Multi-rank runs need one GPU per rank.
    import ctypes as C

    from oracle import oracle as O
    from paper_2511_13061_b200 import macko as M
    from paper_2511_13061_b200.sharded import nccl_sharded_spmv
    from tests.helpers import to_dev, to_host_u16

    class UniqueId(C.Structure):
        _fields_ = [("internal", C.c_char * 128)]

    nccl = C.CDLL("libnccl.so.2")
    uid = UniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    try:
        A = O.gen_dense(2048, 3000, 0.5, 61)
        x = to_dev(O.gen_vector(3000, 62))
        dm = M.DeviceMatrix.from_dense(to_dev(A))
        y = torch.zeros(2048, dtype=torch.float16, device=cuda)
        nccl_sharded_spmv(dm, comm.value, x, y)
        torch.cuda.synchronize()
        assert np.array_equal(to_host_u16(y), to_host_u16(M.spmv(dm, x)))
        with pytest.raises(ValueError):  # slab rows must equal rows_total / ranks
            nccl_sharded_spmv(dm, comm.value, x, torch.zeros(4096, dtype=torch.float16, device=cuda))
    finally:
        nccl.ncclCommDestroy(comm)


def _fused_matrix(R, C):
    """Float-mode test matrix scaled by 2^-4 (exact in fp16) so iterating y = A y stays in range."""
    from oracle import oracle as O

    A = O.gen_dense(R, C, 0.5, 17)
    return (A.view(np.float16) * np.float16(2.0**-4)).astype(np.float16).view(np.uint16)


def _fused_worker(rank, world, port, R, C, out_path):
    # one GPU shared by `world` processes: CUDA IPC between processes on the same device exercises
    # the whole fused all-gather protocol (peer stores, system-scope flags, waits).  The natural
    # loop y = fused(y) runs without any barrier: the double-buffered outputs make it safe.
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2511_13061_b200 import macko as M
        from paper_2511_13061_b200.sharded import FusedRowShardedSpmv, slab_bounds

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        r0, r1 = slab_bounds(R, world, rank)
        A = _fused_matrix(R, C)[r0:r1]
        dm = M.DeviceMatrix.from_dense(torch.from_numpy(A.view(np.int16)).to(dev).view(torch.float16))
        fused = FusedRowShardedSpmv(dm, R, dev)
        y = torch.from_numpy(O.gen_vector(C, 18).view(np.int16)).to(dev).view(torch.float16)
        outs = []
        for step in range(4):
            y = fused(y)
            outs.append(y.clone())  # stream-ordered copy of this step's full y
        torch.cuda.synchronize()
        with pytest.raises(ValueError):
            fused(fused.ys[fused.epoch % 2])  # x overlapping the output buffer is refused
        if rank == 0:
            for step, t in enumerate(outs):
                np.save(out_path + f".{step}.npy", t.view(torch.int16).cpu().numpy().view(np.uint16))
        dist.barrier()
        assert int(fused.flags.cpu().numpy().min()) == 4 * fused.grid
        fused.close()
        dm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_fused_allgather_single_rank(cuda):
    from oracle import oracle as O
    from paper_2511_13061_b200 import macko as M
    from paper_2511_13061_b200.sharded import FusedRowShardedSpmv
    from tests.helpers import b200_y, to_dev, to_host_u16

    A = O.gen_dense(3000, 5000, 0.5, 71)
    x = O.gen_vector(5000, 72)
    dm = M.DeviceMatrix.from_dense(to_dev(A))
    fused = FusedRowShardedSpmv(dm, 3000, cuda)
    ref = b200_y(O.encode_dense(A), x)
    for step in range(1, 4):
        y = fused(to_dev(x))
        torch.cuda.synchronize()
        assert np.array_equal(to_host_u16(y), ref), step
        assert y.data_ptr() == fused.ys[(step - 1) % 2].data_ptr()
        assert int(fused.flags.item()) == step * fused.grid
    fused.close()
    dm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols", [(600, 40000), (3000, 3000), (4099, 700)])
def test_fused_peer_stores_stand_in(cuda, rows, cols):
    # One local buffer stands in for a remote rank's y: rows finished by one warp reach it through
    # the warp's coalesced copy, rows split across warps / CTAs through their last arrival's
    # direct stores, empty rows through the copy of the warp that owns them.
    from oracle import oracle as O
    from paper_2511_13061_b200 import macko as M
    from tests.helpers import b200_y, to_dev, to_host_u16

    A = O.gen_dense(rows, cols, 0.5, 91)
    A[::7] = 0  # empty rows, also at a slab's first and last row
    A[-1] = 0
    x = O.gen_vector(cols, 92)
    dm = M.DeviceMatrix.from_dense(to_dev(A))
    y = torch.zeros(rows, dtype=torch.float16, device=cuda)
    other = [torch.full((rows,), -1.0, dtype=torch.float16, device=cuda) for _ in range(2)]
    flags = torch.zeros(2, dtype=torch.int32, device=cuda)
    dm.set_peers([y.data_ptr(), other[0].data_ptr()], [flags.data_ptr(), flags.data_ptr() + 4])
    dm.set_peer_bank(1, [y.data_ptr(), other[1].data_ptr()])
    ref = b200_y(O.encode_dense(A), x)
    for bank in (0, 1, 0):
        dm.spmv_into(to_dev(x), y, peers=True, bank=bank)
        torch.cuda.synchronize()
        assert np.array_equal(to_host_u16(y), ref)
        assert np.array_equal(to_host_u16(other[bank]), ref), bank
    assert int(flags[0].item()) == int(flags[1].item()) == 3 * dm.launch_info().grid
    dm.set_peers([], [])
    dm.close()


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 4])
def test_fused_allgather_processes_one_gpu(cuda, tmp_path, world):
    # bit-exact against the slab-order oracle: rank g's rows are the kernel order on its own slab
    from oracle import oracle as O
    from paper_2511_13061_b200.sharded import slab_bounds
    from tests.helpers import b200_y

    R = C = 3000
    out = str(tmp_path / "fy")
    mp.spawn(_fused_worker, args=(world, _free_port(), R, C, out), nprocs=world, join=True)
    A = _fused_matrix(R, C)
    slabs = [O.encode_dense(A[a:b]) for a, b in (slab_bounds(R, world, g) for g in range(world))]
    x = O.gen_vector(C, 18)
    for step in range(4):
        x = np.concatenate([b200_y(s, x) for s in slabs])
        assert np.isfinite(x.view(np.float16)).all()
        assert np.array_equal(np.load(out + f".{step}.npy"), x), step


def _fused_chain_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_13061_b200 import decoder_chain as D
        from paper_2511_13061_b200 import macko as M

        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        # density 1: every row starts at a multiple of 8 in the slabs and in the whole matrices,
        # so the sharded chain is bit-identical to the unsharded one
        shape = D.ChainShape(layers=2, hidden=256, inter=688)
        ch = D.SparseDecoderChain(shape, density=1.0, seed=5, device=dev, fused=True)
        M.gen_vector(ch.acts["h"], 256, seed=6)
        ch.acts["h"].mul_(2.0**-8)
        for tok in range(2):
            ch.forward_token(pdl=bool(tok))
            torch.cuda.synchronize()
            dist.barrier()
        np.save(out_path + f".{rank}.npy", ch.acts["h"].view(torch.int16).cpu().numpy().view(np.uint16))
        ch.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_fused_decode_chain_two_processes_one_gpu(cuda, tmp_path):
    from paper_2511_13061_b200 import decoder_chain as D
    from paper_2511_13061_b200 import macko as M

    out = str(tmp_path / "chain")
    mp.spawn(_fused_chain_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    shape = D.ChainShape(layers=2, hidden=256, inter=688)
    ref = D.SparseDecoderChain(shape, density=1.0, seed=5)
    M.gen_vector(ref.acts["h"], 256, seed=6)
    ref.acts["h"].mul_(2.0**-8)
    for _ in range(2):
        ref.forward_token(pdl=False)
    torch.cuda.synchronize()
    want = ref.acts["h"].view(torch.int16).cpu().numpy().view(np.uint16)
    for r in range(2):
        assert np.array_equal(np.load(out + f".{r}.npy"), want), r
    ref.close()
