"""Host-side logic of the multi-GPU path on CPU (gloo, world size 2 and 4): the z-slab /
y-slab decomposition with the block all-to-all S[r][s] -> R[s][r] of DESIGN.md §9 reproduces
the single-domain Galerkin projection and preconditioner of the oracle, including the
rank-local ky offset of the frequency symbol and the rank-0 zero frequency.

This is a NumPy emulation of the slab algorithm (test infrastructure); the CUDA/NCCL
implementation of the same layout is checked on one GPU by test_gpu_ops::
test_emulated_slab_layout (FGD_EMULATE_SLABS)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.projection import apply_projection, project_spectrum
from oracle.spectral import Grid

N = (8, 8, 8)
MASK = (1, 1, 0, 1, 1, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _all_to_all(out, inp):
    """block all-to-all with point-to-point messages (gloo has no alltoall): out[p] <- inp[rank] of p."""
    rank, P = dist.get_rank(), dist.get_world_size()
    reqs = []
    for p in range(P):
        if p == rank:
            out[p].copy_(inp[p])
        else:
            reqs.append(dist.isend(inp[p], p))
            reqs.append(dist.irecv(out[p], p))
    for r in reqs:
        r.wait()


def _slab_projection(rank, P, tau_local, g):
    """tau_local: (6, nz_l, Ny, Nx) real slab of rank r.  Returns the slab of G*(tau)."""
    Nx, Ny, Nz = g.n
    nzs, nys, Hx = Nz // P, Ny // P, Nx // 2 + 1
    # x (R2C) and y (C2C) transforms are slab-local
    A = np.fft.fft(np.fft.rfft(tau_local, axis=-1), axis=-2)          # (6, nzs, Ny, Hx)
    # pack S[s] = (6, Hx, nys, nzs) for every destination y-slab s
    send = [np.ascontiguousarray(np.transpose(A[:, :, s * nys:(s + 1) * nys, :], (0, 3, 2, 1))) for s in range(P)]
    recv = [np.empty_like(send[0]) for _ in range(P)]
    ts = [torch.from_numpy(np.stack([x.real, x.imag])) for x in send]
    tr = [torch.empty_like(ts[0]) for _ in range(P)]
    _all_to_all(tr, ts)
    for p in range(P):
        recv[p] = tr[p][0].numpy() + 1j * tr[p][1].numpy()
    # R: full z lines for the local ky rows: concatenate source z-slabs
    R = np.concatenate(recv, axis=-1)                                  # (6, Hx, nys, Nz)
    Rz = np.fft.fft(R, axis=-1)
    # global frequency symbol for kx in [0, Hx), ky in this rank's y-slab, kz in [0, Nz)
    k = g.symbol(half=True)                                            # (3, Nz, Ny, Hx)
    kloc = np.transpose(k[:, :, rank * nys:(rank + 1) * nys, :], (0, 3, 2, 1))   # (3, Hx, nys, Nz)
    flat = Rz.reshape(6, -1)
    kf = kloc.reshape(3, -1)
    has_dc = rank == 0
    if has_dc:
        out = project_spectrum(flat, kf, MASK, dc_index=(0,))
    else:
        out = project_spectrum(np.concatenate([np.zeros((6, 1)), flat], 1), np.concatenate([np.zeros((3, 1)), kf], 1),
                               MASK, dc_index=(0,))[:, 1:]
    Ri = np.fft.ifft(out.reshape(Rz.shape), axis=-1)
    back = [np.ascontiguousarray(Ri[..., p * nzs:(p + 1) * nzs]) for p in range(P)]
    tb = [torch.from_numpy(np.stack([x.real, x.imag])) for x in back]
    tr2 = [torch.empty_like(tb[0]) for _ in range(P)]
    _all_to_all(tr2, tb)
    A2 = np.empty_like(A)
    for s in range(P):
        blk = tr2[s][0].numpy() + 1j * tr2[s][1].numpy()              # (6, Hx, nys, nzs)
        A2[:, :, s * nys:(s + 1) * nys, :] = np.transpose(blk, (0, 3, 2, 1))
    return np.fft.irfft(np.fft.ifft(A2, axis=-2), n=Nx, axis=-1)


def _worker(rank, P, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        g = Grid(N, (1.0, 1.0, 1.0))
        tau = np.random.default_rng(3).normal(size=(6,) + g.shape)
        nzs = g.n[2] // P
        y = _slab_projection(rank, P, tau[:, rank * nzs:(rank + 1) * nzs], g)
        ref = apply_projection(g, tau, MASK)[:, rank * nzs:(rank + 1) * nzs]
        q.put((rank, float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 4])
def test_slab_projection_matches_single_domain(P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    res = [q.get(timeout=60) for _ in range(P)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err < 1e-12, (rank, err)
