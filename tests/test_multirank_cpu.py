"""World-size-2/3 CPU tests (gloo) of the multi-GPU host logic: row-block shards, the halo
plan of libigs (igs_plan_ghosts / igs_plan_remap), the request exchange igs_create performs
with NCCL (here with gloo send/recv), and the invariant it relies on: the sharded SpMV with
halo equals the global SpMV bitwise, and the per-rank partial dots summed by an allreduce
equal the global dots.  The shard bounds are bench.py's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_2205_07805_b200 as P
        import workloads as W
        import bench

        n = N ** 3
        bench_N = bench.N_GRID
        bench.N_GRID = N                    # reuse bench.py's plane-aligned shard bounds
        bounds = np.array([bench.shard_bounds(n, world, r)[0] for r in range(world)] + [n])
        bench.N_GRID = bench_N
        r0, r1 = bounds[rank], bounds[rank + 1]
        A = W.stencil_csr(N, 3, W.C4_BETA, r0, r1)
        ghosts, cnt = P.igs_plan_ghosts(r0, A.n_rows, A.rowptr, A.colind, world, bounds)
        # count matrix (igs_create: ncclAllGather)
        allc = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, torch.from_numpy(cnt))
        allc = torch.stack(allc).numpy()
        # request exchange (igs_create: ncclSend/ncclRecv of global indices)
        reqs, ops = {}, []
        off = 0
        for peer in range(world):
            rc = int(allc[rank, peer]); sc = int(allc[peer, rank])
            if peer != rank and rc:
                ops.append(dist.isend(torch.from_numpy(ghosts[off:off + rc].copy()), peer))
            if peer != rank and sc:
                reqs[peer] = torch.zeros(sc, dtype=torch.int64)
                ops.append(dist.irecv(reqs[peer], peer))
            off += rc if peer != rank else 0
        for o in ops:
            o.wait()
        send_idx = {pr: t.numpy() - r0 for pr, t in reqs.items()}
        for pr, idx in send_idx.items():
            assert idx.min() >= 0 and idx.max() < A.n_rows
        # one iteration's halo + SpMV on a seeded vector
        x = np.random.default_rng(5).standard_normal(n)
        xl = x[r0:r1]
        ghost_vals = np.zeros(ghosts.size)
        ops, recv_bufs = [], {}
        off = 0
        for peer in range(world):
            rc = int(allc[rank, peer])
            if peer in send_idx:
                ops.append(dist.isend(torch.from_numpy(xl[send_idx[peer]].copy()), peer))
            if peer != rank and rc:
                recv_bufs[peer] = (off, torch.zeros(rc, dtype=torch.float64))
                ops.append(dist.irecv(recv_bufs[peer][1], peer))
            off += rc if peer != rank else 0
        for o in ops:
            o.wait()
        for peer, (o0, t) in recv_bufs.items():
            ghost_vals[o0:o0 + t.numel()] = t.numpy()
        np.testing.assert_array_equal(ghost_vals, x[ghosts])
        loc = P.igs_plan_remap(r0, A.n_rows, A.rowptr, A.colind, ghosts)
        Aloc = W.Csr(A.n_rows, A.n_rows + ghosts.size, 0, A.rowptr, loc, A.values)
        y_loc = oracle.spmv(Aloc, np.concatenate([xl, ghost_vals]))
        # partial dots + allreduce (the single synchronisation)
        Vb = np.random.default_rng(9).standard_normal((n, 4))
        part = torch.from_numpy(oracle.block_dot(Vb[r0:r1], xl, y_loc, block=0))
        dist.all_reduce(part)
        ys = [None] * world                   # uneven shards: gather as objects
        dist.all_gather_object(ys, y_loc)
        if rank == 0:
            y = np.concatenate(ys)
            Ag = W.stencil_csr(N, 3, W.C4_BETA)
            y_ref = oracle.spmv(Ag, x)
            assert y.tobytes() == y_ref.tobytes()           # bitwise: same row order
            ref = oracle.block_dot(Vb, x, y_ref, block=0)
            assert np.allclose(part.numpy(), ref, rtol=1e-12, atol=1e-10)
        # unique-id broadcast as bench.py does it (128 bytes)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world,N", [(2, 12), (3, 10)])
def test_sharded_spmv_and_reduction_gloo(world, N):
    from paper_2205_07805_b200 import build
    build.build()
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r, msg in out:
        assert msg == "ok", f"rank {r}: {msg}"


def _alg3_worker(rank, world, port, N, k, q):
    """Row-partitioned Alg. 3 exactly as libigs distributes it: every rank owns a row block
    of A, V and the vectors; per iteration one halo exchange (SpMV ghosts) and ONE allreduce
    of the 2(p+1) partial dots; the small step is replicated on every rank from the reduced
    vector.  Written here in numpy (test scaffolding) to pin the distribution scheme against
    the oracle's single-process Alg. 3."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_2205_07805_b200 as P
        import workloads as W
        n = N ** 3
        bounds = np.array([n * r // world for r in range(world)] + [n])
        r0, r1 = bounds[rank], bounds[rank + 1]
        prob = W.config("c4", N=N, row_begin=r0, row_end=r1)
        A, b = prob.A, prob.b
        ghosts, cnt = P.igs_plan_ghosts(r0, A.n_rows, A.rowptr, A.colind, world, bounds)
        loc = P.igs_plan_remap(r0, A.n_rows, A.rowptr, A.colind, ghosts)
        Aloc = W.Csr(A.n_rows, A.n_rows + ghosts.size, 0, A.rowptr, loc, A.values)
        nallred = [0]

        def allreduce(v):
            t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
            dist.all_reduce(t)
            nallred[0] += 1
            return t.numpy()

        def spmv(xl):   # halo: gather every rank's block (scaffolding), take the ghosts
            parts = [None] * world
            dist.all_gather_object(parts, xl)
            xg = np.concatenate(parts)
            return oracle.spmv(Aloc, np.concatenate([xl, xg[ghosts]]))

        m = k
        V = np.zeros((A.n_rows, m + 1)); H = np.zeros((m + 1, m)); HP = np.zeros((m + 1, m))
        L = np.zeros((m, m))
        rho = np.sqrt(allreduce([b @ b])[0])
        V[:, 0] = b / rho
        z = spmv(V[:, 0])
        h = allreduce([V[:, 0] @ z])[0]
        HP[0, 0] = h
        V[:, 1] = z - h * V[:, 0]
        per_iter = []
        for p in range(1, m + 1):
            u = V[:, p]
            a0 = nallred[0]
            drain = p == m
            if not drain:
                z = spmv(u)
            loc_d = np.concatenate([V[:, :p].T @ u, [u @ u]] + ([] if drain else [V[:, :p].T @ z, [u @ z]]))
            dv = allreduce(loc_d)                         # the single synchronisation
            per_iter.append(nallred[0] - a0)
            r2, s = dv[:p], dv[p]
            r3 = oracle.forward_solve_unit(L[:p, :p], r2)
            gamma = np.sqrt(s - r2 @ r2)
            H[:p, p - 1] = HP[:p, p - 1] + r3
            H[p, p - 1] = gamma
            V[:, p] = (u - V[:, :p] @ r2) / gamma
            if drain:
                break
            c, d = dv[p + 1:2 * p + 1] / gamma, dv[2 * p + 1] / gamma ** 2
            L[p, :p] = r2 / gamma
            r1 = np.concatenate([c, [d - L[p, :p] @ c]])
            V[:, p + 1] = z / gamma - V[:, :p + 1] @ r1
            HP[:p + 1, p] = r1 - H[:p + 1, :p] @ (r2 / gamma)
        assert all(c == 1 for c in per_iter), per_iter
        if rank == 0:
            Pg = W.config("c4", N=N)
            o = oracle.gmres(Pg.A, Pg.b, k, variant="igs2")
            d = oracle.column_normwise_diff(H, o["H"], k)
            assert d <= 1e-10, d
        H_all = [None] * world
        dist.all_gather_object(H_all, H)
        for Hr in H_all:                                   # replicated state is bit-identical
            assert Hr.tobytes() == H_all[0].tobytes()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_alg3_one_allreduce_per_iteration_gloo(world):
    from paper_2205_07805_b200 import build
    build.build()
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_alg3_worker, args=(r, world, port, 8, 24, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r, msg in out:
        assert msg == "ok", f"rank {r}: {msg}"
