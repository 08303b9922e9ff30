"""Multi-GPU slice sharding, host side, on CPU.

* sacd_shard_plan (libsacd, pure host code) partitions every mode's nonzeros into
  nnz-balanced ranges and every row to exactly one owner, for any world size.
* The exchange protocol the library runs over NCCL is emulated here with world_size 2
  and 3 gloo process groups, with the fp64 oracle doing the compute: each rank computes
  the MTTKRP of its own nonzero range, head partials are all-gathered and added by the
  row owners in rank order, owners run the row pass on their rows, the updated rows are
  all-gathered, Grams / ti / E are reduced in rank order.  The result must equal the
  unsharded oracle run (same decisions, same branch, f to 1e-12).
* The peer-memory exchange (exchange "p2p": changed 16-byte chunks stored into every peer's
  replica, device flags) is emulated with per-rank replicas, which must stay bitwise
  identical.
* The delta exchange is emulated the same way: each owner lists the elements of
  its rows that changed bit for bit (flat index, value), the list lengths are all-gathered
  and every rank takes the lists when they are smaller than the rows (12 vs 8 bytes per
  element), else the rows; the others apply the lists.  Same result as the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import sacd_inputs as SI


@pytest.fixture(scope="module")
def plan():
    from paper_2003_03572_b200 import build, sacd
    build.build()
    return sacd.shard_plan


def random_row_ptr(I, seed, heavy=()):
    rng = np.random.default_rng(seed)
    counts = rng.poisson(3.0, size=I)
    counts[rng.random(I) < 0.3] = 0                        # empty rows
    for r, c in heavy:
        counts[r] = c
    return np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_plan_partitions_rows_and_nonzeros(plan, world, case):
    if case == 0:
        rp = random_row_ptr(100, 1)
    elif case == 1:
        rp = random_row_ptr(50, 2, heavy=((0, 500), (7, 300), (49, 800)))   # rows spanning ranks
    elif case == 2:
        rp = np.zeros(11, np.int64)                                          # empty tensor
    else:
        rp = np.array([0, 0, 0, 1000, 1000], np.int64)                       # one row holds everything
    I, nnz = len(rp) - 1, int(rp[-1])
    plans = [plan(rp, world, p) for p in range(world)]
    owner = np.full(I, -1)
    for p, (lo, hi, rlo, rhi, head) in enumerate(plans):
        assert lo == p * nnz // world and hi == (p + 1) * nnz // world
        assert (owner[rlo:rhi] == -1).all()
        owner[rlo:rhi] = p
        for r in range(rlo, rhi):
            assert lo <= rp[r] < hi or (rp[r] == nnz and p == world - 1) or (rp[r] == hi and rp[r] == rp[r + 1] and p == world - 1)
        if head >= 0:
            assert rp[head] < lo < rp[head + 1]
            assert owner[head] != -1 and owner[head] < p
    assert (owner >= 0).all()
    # every nonzero is counted exactly once: owner's local part + heads of higher ranks
    for r in range(I):
        q = owner[r]
        lo, hi = plans[q][0], plans[q][1]
        got = max(0, min(rp[r + 1], hi) - max(rp[r], lo))
        for p2, (lo2, hi2, rlo2, rhi2, head2) in enumerate(plans):
            if head2 == r:
                assert p2 > q
                got += min(rp[r + 1], hi2) - lo2
        assert got == rp[r + 1] - rp[r]


# ----------------------------------------------------------------------------- gloo emulation
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, K, q, exchange="rows"):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2003_03572_b200 import sacd
        dims, R, seed = (40, 30, 20), 4, 3
        c, v = SI.tiny_tensor(dims, 0.08, 5)
        c, v = c.numpy(), v.numpy()
        # make a heavy slice so rows span ranks
        F = O.init_factors(dims, R, seed)
        lay = [O.layout(c, v, dims, n) for n in range(3)]
        plans = [[sacd.shard_plan(lay[n][3], world, p) for p in range(world)] for n in range(3)]
        zp = [np.zeros((dims[n], R)) for n in range(3)]
        hist = [[], [], []]
        fs, Es, brs = [], [], []
        used_delta = [0]
        xn2 = float((v.astype(np.float64) ** 2).sum())
        for k in range(1, K + 1):
            Erow, brrow, mdot = [], [], 0.0
            for n in range(3):
                a, b = O.other_modes(dims, n)
                ia, ib, vv, rp = lay[n]
                lo, hi, rlo, rhi, head = plans[n][rank]
                # (1) local MTTKRP over the nonzero range [lo, hi): clipped row_ptr
                rpl = np.clip(rp, lo, hi)
                M = O.mttkrp_layout(rpl, ia, ib, vv, F[a], F[b])
                # (2) head partials all-gathered, added by the owner in rank order
                send = torch.zeros(R + 1, dtype=torch.float64)
                send[0] = head
                if head >= 0:
                    send[1:] = torch.from_numpy(M[head])
                recv = [torch.zeros(R + 1, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(recv, send)
                for p2 in range(world):
                    h = int(recv[p2][0])
                    if rlo <= h < rhi:
                        M[h] += recv[p2][1:].numpy()
                # (3) H from the replicated factors' Grams; the branch from the shared history
                H = O.hadamard(O.gram(F[a]), O.gram(F[b]))
                br = O.branch(k, hist[n])
                Fn, zn, ti, E, Ech, md, _ = O.mode_pass(M[rlo:rhi], H, F[n][rlo:rhi], zp[n][rlo:rhi], br)
                zp[n][rlo:rhi] = zn
                # (4) updated rows all-gathered into the replicated factor
                if exchange == "p2p":
                    # peer-memory exchange: every 16-byte chunk (2 fp64) of the owned rows that
                    # changed against the pass-start snapshot is stored into every peer's
                    # replica; the all-gather stands for the stores + the flag barrier
                    old = F[n][rlo:rhi].copy()
                    F[n][rlo:rhi] = Fn
                    a_new = F[n][rlo:rhi].reshape(-1, 2).view(np.int64)
                    a_old = old.reshape(-1, 2).view(np.int64)
                    ch = np.nonzero((a_new != a_old).any(axis=1))[0]
                    msg = (ch + rlo * R // 2, F[n][rlo:rhi].reshape(-1, 2)[ch].copy())
                    msgs = [None] * world
                    dist.all_gather_object(msgs, msg)
                    chunks = F[n].reshape(-1, 2)
                    for p2, (ix, vals) in enumerate(msgs):
                        if p2 != rank:
                            chunks[ix] = vals
                    used_delta[0] += 1
                elif exchange == "delta":
                    old = F[n][rlo:rhi]
                    ch = (Fn.view(np.int64) != old.view(np.int64)).reshape(-1)
                    idx = np.nonzero(ch)[0] + rlo * R
                    lst = (idx.astype(np.uint32), Fn.reshape(-1)[ch].copy())
                    cnt = torch.tensor([len(idx)], dtype=torch.int64)
                    cnts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
                    dist.all_gather(cnts, cnt)
                    nd = int(sum(int(x) for x in cnts))
                    nfull = sum((plans[n][p2][3] - plans[n][p2][2]) * R for p2 in range(world))
                    F[n][rlo:rhi] = Fn
                    if nd * 12 < nfull * 8:
                        lists = [None] * world
                        dist.all_gather_object(lists, lst)
                        flat = F[n].reshape(-1)
                        for p2, (ix, vals) in enumerate(lists):
                            assert len(ix) == int(cnts[p2])
                            if p2 != rank:
                                flat[ix.astype(np.int64)] = vals
                        used_delta[0] += 1
                    else:
                        rows = [None] * world
                        dist.all_gather_object(rows, (rlo, rhi, Fn))
                        for (r0, r1, blk) in rows:
                            F[n][r0:r1] = blk
                else:
                    rows = [None] * world
                    dist.all_gather_object(rows, (rlo, rhi, Fn))
                    for (r0, r1, blk) in rows:
                        F[n][r0:r1] = blk
                # (5) scalars reduced in rank order
                sc = [None] * world
                dist.all_gather_object(sc, (ti, E, md))
                ti_t = 0.0
                E_t = 0
                md_t = 0.0
                for (t_, e_, m_) in sc:
                    ti_t += t_
                    E_t += e_
                    md_t += m_
                hist[n].append(ti_t)
                Erow.append(E_t)
                brrow.append(br)
                if n == 2:
                    mdot = md_t
            G = [O.gram(F[n]) for n in range(3)]
            fs.append(xn2 - 2 * mdot + float((G[0] * G[1] * G[2]).sum()))
            Es.append(Erow)
            brs.append(brrow)
        reps = [None] * world
        dist.all_gather_object(reps, [x.copy() for x in F])
        same = all(np.array_equal(reps[p2][n], reps[0][n]) for p2 in range(world) for n in range(3))
        if rank == 0:
            q.put((fs, Es, brs, [x.copy() for x in F], used_delta[0], same))
        dist.destroy_process_group()
    except Exception as ex:  # surface worker failures to the parent
        q.put(("error", repr(ex)))
        raise


@pytest.mark.parametrize("world,exchange", [(2, "rows"), (3, "rows"), (2, "delta"), (3, "delta"), (2, "p2p"),
                                            (3, "p2p")])
def test_sharded_sweeps_equal_unsharded_oracle(plan, world, exchange):
    K = 6 if exchange != "rows" else 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert res[0] != "error", res
    fs, Es, brs, F, used, same = res
    assert same  # every rank's replica is bitwise identical
    if exchange != "rows":
        assert used > 0
    dims, R, seed = (40, 30, 20), 4, 3
    c, v = SI.tiny_tensor(dims, 0.08, 5)
    ora = O.sacd_run(c.numpy(), v.numpy(), dims, R, seed, K)
    np.testing.assert_allclose(fs, ora["f"][1:], rtol=1e-12)
    assert np.array_equal(np.array(Es), ora["E"])
    assert np.array_equal(np.array(brs), ora["branch"])
    for n in range(3):
        np.testing.assert_allclose(F[n], ora["F"][n], rtol=1e-10, atol=1e-13)
