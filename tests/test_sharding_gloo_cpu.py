"""CPU, world_size = 2 over gloo: the row-sharded protocol of the multi-GPU path (SURVEY.md 5.8,
C1/C2/C3/C5 and the point-cloud maximum) -- what each rank reduces locally, what crosses the wire, and how the pieces are combined --
checked against the unsharded oracle.  Per-rank kernel work is stood in by the oracle on the rank's row
block; the partition and the threshold search are the product's own host functions
(regot_b200_host_row_block / regot_b200_host_pick_bucket, also used by the device path)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_08793_b200 import _lib
from tests import oracle_lib

WORLD = 2


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def row_block(n, rank, world):
    b, c = C.c_int64(), C.c_int64()
    _lib.load().regot_b200_host_row_block(n, rank, world, C.byref(b), C.byref(c))
    return b.value, c.value


def pick_bucket(hist, need):
    h = np.ascontiguousarray(hist, dtype=np.uint64)
    b, above = C.c_int(), C.c_int64()
    _lib.load().regot_b200_host_pick_bucket(h.ctypes.data_as(C.POINTER(C.c_uint64)), len(h), need, C.byref(b), C.byref(above))
    return b.value, above.value


def allreduce(x, op=dist.ReduceOp.SUM):
    t = torch.from_numpy(np.ascontiguousarray(x).copy())
    dist.all_reduce(t, op=op)
    return t.numpy()


def order_key(T):
    T = T + 0.0
    bits = T.view(np.uint64)
    neg = (bits >> np.uint64(63)).astype(bool)
    return np.where(neg, ~bits, bits | np.uint64(1 << 63))


def sharded_gradient(o, p, al, be, rank):
    n, m = p["n"], p["m"]
    r0, cnt = row_block(n, rank, WORLD)
    blk = dict(n=cnt, m=m, M=np.asfortranarray(p["M"][r0:r0 + cnt]), a=p["a"][r0:r0 + cnt], b=p["b"], eta=p["eta"])
    g = o.gradient(blk, al[r0:r0 + cnt], be)
    ga = g["row"] - blk["a"]
    # C1 payload: local column sums + row-side scalars (k1_gradient.cu: pack[m + k])
    pack = np.concatenate([g["col"], [g["row"].sum(), al[r0:r0 + cnt] @ blk["a"], np.abs(ga).sum(), al[r0:r0 + cnt] @ ga, ga @ ga]])
    pack = allreduce(pack)
    col, S = pack[:m], pack[m:]
    gb = col - p["b"]
    f = p["eta"] * S[0] - S[1] - be[:m - 1] @ p["b"][:m - 1]
    return dict(f=f, col=col, marginal_error=S[2] + np.abs(gb).sum(), gap=S[3] + be @ gb,
                grad_norm2=np.sqrt(S[4] + gb[:m - 1] @ gb[:m - 1]), row=g["row"], r0=r0)


def sharded_optimal_beta(p, al, rank):
    n, m, eta = p["n"], p["m"], p["eta"]
    r0, cnt = row_block(n, rank, WORLD)
    v = (al[r0:r0 + cnt, None] - p["M"][r0:r0 + cnt]) / eta
    loc_max = v.max(axis=0)
    loc_sum = np.exp(v - loc_max).sum(axis=0)
    glob_max = allreduce(loc_max, dist.ReduceOp.MAX)          # C2: allreduce(MAX) of the maxima ...
    glob_sum = allreduce(loc_sum * np.exp(loc_max - glob_max))  # ... rescale, allreduce(SUM)
    return eta * (np.log(p["b"]) - (glob_max + np.log(glob_sum)))


def sharded_topk(T, k, rank):
    n, m = T.shape
    mm1 = m - 1
    r0, cnt = row_block(n, rank, WORLD)
    key = order_key(np.ascontiguousarray(T[r0:r0 + cnt, :mm1]))
    rows, cols = np.meshgrid(np.arange(r0, r0 + cnt), np.arange(mm1), indexing="ij")
    take = min(k, n * mm1)
    star = (rows == 0) | (cols == 0)
    keep = star.copy()
    if take > 0:
        hist = allreduce(np.bincount((key >> np.uint64(52)).astype(np.int64).ravel(), minlength=4096).astype(np.int64))
        bstar, above = pick_bucket(hist, take)
        rem = take - above
        fixed_mask, fixed_val = np.uint64(0xFFF << 52), np.uint64(bstar << 52)
        for shift in (39, 26, 13, 0):
            sel = (key & fixed_mask) == fixed_val
            digit = ((key[sel] >> np.uint64(shift)) & np.uint64(8191)).astype(np.int64)
            h = allreduce(np.bincount(digit, minlength=8192).astype(np.int64))
            d, above = pick_bucket(h, rem)
            rem -= above
            fixed_mask |= np.uint64(8191 << shift)
            fixed_val |= np.uint64(d << shift)
        kstar, need_eq = fixed_val, rem
        tie = key == kstar
        counts = np.zeros(WORLD, np.int64)
        counts[rank] = tie.sum()
        counts = allreduce(counts)
        offset = counts[:rank].sum()
        tie_rank = np.cumsum(tie.ravel()).reshape(tie.shape) - 1  # row-major order inside the block
        keep |= (key > kstar) | (tie & (offset + tie_rank < need_eq))
    coords = np.stack([rows[keep], cols[keep]], axis=1).astype(np.int32)
    gathered = [None] * WORLD
    dist.all_gather_object(gathered, coords)
    return np.concatenate(gathered)  # rank order == row order


def sharded_schur_pcg(B, D1, D2, ra, rb, rank, rtol=1e-12, max_iter=500):
    """The kernel-by-kernel Schur-complement PCG of k4_sparse.cu (pcg_schur_multikernel) on a row block:
    alpha-space quantities and the rows of B are local, beta-space vectors are replicated, and the ONLY
    collectives are one allreduce(SUM) of B' t per mat-vec plus the alpha part of the reference norm."""
    n = B.shape[0]
    r0, cnt = row_block(n, rank, WORLD)
    Bl, D1l, ral = B[r0:r0 + cnt], D1[r0:r0 + cnt], ra[r0:r0 + cnt]
    t = ral / D1l
    g0 = allreduce(np.array([ral @ t]))[0] + rb @ (rb / D2)     # r' D^-1 r of the FULL system
    u = allreduce(Bl.T @ t)                                       # C3: the one vector collective
    r = rb - u
    z = r / D2
    p, x = z.copy(), np.zeros_like(rb)
    rz = r @ z
    its = 0
    while rz > rtol * rtol * g0 and its < max_iter:
        t = (Bl @ p) / D1l
        u = allreduce(Bl.T @ t)
        q = D2 * p - u
        a = rz / (p @ q)                                           # beta-space dots: identical on every rank
        x += a * p
        r -= a * q
        z = r / D2
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
        its += 1
    xa = ral / D1l - (Bl @ x) / D1l
    return xa, x, its, r0


def sharded_cloud_max(X, Y, rank):
    """regot_b200_set_pointcloud_rows: the normalising maximum is taken over all ranks (allreduce MAX)."""
    r0, cnt = row_block(X.shape[0], rank, WORLD)
    d2 = ((X[r0:r0 + cnt, None, :] - Y[None, :, :]) ** 2).sum(axis=2)
    return allreduce(np.array([d2.max()]), dist.ReduceOp.MAX)[0]


def worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        o = oracle_lib.load()
        res = {}
        for tag, (kind, n, m, eta) in {"g1": ("rand", 37, 29, 0.1), "g2": ("synth2", 64, 50, 0.001)}.items():
            p = o.gen_problem(kind, n, m, eta, seed=11)
            al, be = o.rand_dual(n, m, 0.05, 12)
            s, ref = sharded_gradient(o, p, al, be, rank), o.gradient(p, al, be)
            np.testing.assert_allclose(s["col"], ref["col"], rtol=1e-13)
            np.testing.assert_allclose(s["row"], ref["row"][s["r0"]:s["r0"] + len(s["row"])], rtol=1e-13)
            assert abs(s["f"] - ref["f"]) <= 1e-12 * (1 + abs(ref["f"]))
            assert abs(s["marginal_error"] - ref["marginal_error"]) <= 1e-12 * (1 + ref["marginal_error"])
            assert abs(s["gap"] - ref["duality_gap"]) <= 1e-12 * (1 + abs(ref["duality_gap"]))
            assert abs(s["grad_norm2"] - ref["grad_norm2"]) <= 1e-12 * (1 + ref["grad_norm2"])
            b = sharded_optimal_beta(p, al, rank)
            np.testing.assert_allclose(b, o.optimal_beta(p, al), rtol=0, atol=1e-13 * max(1.0, np.abs(b).max()))
            res[tag] = True
        rng = np.random.default_rng(5)  # same stream on both ranks
        for t in range(6):
            n, m = int(3 + rng.random() * 40), int(3 + rng.random() * 40)
            T = np.where(rng.random((n, m)) < 0.3, 0.5, rng.random((n, m)))  # injected ties across the shard boundary
            k = int(rng.random() * n * (m - 1))
            got = sharded_topk(T, k, rank)
            want = o.select_topk(T, k)
            assert np.array_equal(got, want), (t, n, m, k)
        got = sharded_topk(T, 0, rank)
        assert np.array_equal(got, o.select_topk(T, 0))
        # Schur-complement PCG over row blocks == dense solve of A = [D1 B; B' D2]
        n, m = 41, 23
        B = np.where(rng.random((n, m)) < 0.3, rng.random((n, m)), 0.0)
        D1, D2 = B.sum(axis=1) + 0.5 + rng.random(n), B.sum(axis=0) + 0.5 + rng.random(m)  # diagonally dominant: SPD
        ra, rb = rng.normal(size=n), rng.normal(size=m)
        xa, xb, its, r0 = sharded_schur_pcg(B, D1, D2, ra, rb, rank)
        A = np.block([[np.diag(D1), B], [B.T, np.diag(D2)]])
        ref = np.linalg.solve(A, np.concatenate([ra, rb]))
        assert 0 < its < 200
        np.testing.assert_allclose(xa, ref[r0:r0 + len(xa)], rtol=0, atol=1e-10 * np.abs(ref).max())
        np.testing.assert_allclose(xb, ref[n:], rtol=0, atol=1e-10 * np.abs(ref).max())
        # point clouds: global maximum of the cost
        X, Y = rng.normal(size=(19, 3)), rng.normal(size=(11, 3))
        assert sharded_cloud_max(X, Y, rank) == ((X[:, None, :] - Y[None, :, :]) ** 2).sum(axis=2).max()
        out[rank] = True
    finally:
        dist.destroy_process_group()


def test_row_sharded_protocol_world2():
    port = free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(worker, args=(port, out), nprocs=WORLD, join=True)
        assert dict(out) == {0: True, 1: True}
