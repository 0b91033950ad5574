"""World-size-2 gloo test (CPU) of the rank-local exchange: the NCCL
transport's all-to-all-v descriptors (holder-major send slots, owner-major
receive slots, scheduler.py:244-252 entry order) deliver every holder row to
its owner in ascending sender order, and back (push-from-owner)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.split_oracle import split_sample


class _Meta:
    pass


class _FakeSplit:
    """host_meta() computed from the oracle plan (the same formulas as the
    device splitter's k_pair_scan)."""

    def __init__(self, plan, g, L):
        m = _Meta()
        m.cnt = np.zeros((L + 1, g, g), dtype=np.int64)
        for (l, s, o), e in plan.items():
            m.cnt[l, s, o] = len(e[0])
        m.ref_off = np.zeros((L + 1, g + 1), dtype=np.int64)
        m.recv_off = np.zeros((L + 1, g + 1), dtype=np.int64)
        for l in range(L + 1):
            m.ref_off[l, 1:] = np.cumsum(m.cnt[l].sum(axis=1))
            m.recv_off[l, 1:] = np.cumsum(m.cnt[l].sum(axis=0))
        self.m = m

    def host_meta(self):
        return self.m


def _case():
    rng = np.random.default_rng(0)
    n, g = 400, 2
    V0 = rng.permutation(n)[:120]
    V1 = V0[:40]
    src = rng.integers(0, 120, 300)
    dst = rng.integers(0, 40, 300)
    src = np.r_[np.arange(40), src]
    dst = np.r_[np.arange(40), dst]
    asn = rng.integers(0, g, n)
    splits, plan = split_sample([V0, V1], [(src, dst)], asn, g)
    return splits, plan, g


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_13775_b200.exchange import NcclTransport
        splits, plan, g = _case()
        fake = _FakeSplit(plan, g, 1)
        m = fake.m
        l, stride = 1, 3
        P = int(m.ref_off[l, g])
        # holder-major pair layout: rows = (gid, holder, owner)
        send = torch.zeros((P, stride))
        for (ll, s, o), (gids, hidx, oidx) in sorted(plan.items()):
            if s != rank:
                continue
            base = m.ref_off[l, s] + m.cnt[l, s, :o].sum()
            for j, gid in enumerate(gids):
                send[base + j] = torch.tensor([gid, s, o], dtype=torch.float32)
        recv = torch.full((P, stride), -1.0)
        tr = NcclTransport(rank, world)
        tr.to_owner(fake, l, send, recv, stride)
        r0, r1 = int(m.recv_off[l, rank]), int(m.recv_off[l, rank + 1])
        got = recv[r0:r1].numpy()
        want = []
        for s in range(g):  # ascending sender, then the entry's gid order
            e = plan.get((l, s, rank))
            if e is not None:
                want += [[gid, s, rank] for gid in e[0]]
        ok1 = np.array_equal(got, np.asarray(want, dtype=np.float32).reshape(-1, stride))
        # push-from-owner: owner echoes rows back, holders get them in pair layout
        back = torch.full((P, stride), -1.0)
        tr.from_owner(fake, l, recv, back, stride)
        s0, s1 = int(m.ref_off[l, rank]), int(m.ref_off[l, rank + 1])
        ok2 = np.array_equal(back[s0:s1].numpy(), send[s0:s1].numpy())
        t = torch.full((5,), float(rank + 1))
        tr.all_reduce(t)
        ok3 = bool(torch.all(t == 3.0))
        q.put((rank, ok1, ok2, ok3))
    finally:
        dist.destroy_process_group()


def test_nccl_transport_descriptors_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 2000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] and r[2] and r[3] for r in res), res
