"""Transports for the push-to-owner / push-from-owner rounds.

LocalTransport: all g devices live in this process (one GPU): one copy kernel
per round moves every holder->owner block (the reference's in-process
exchange, engine.py:125-156, without the Python loops).

NcclTransport: one process per GPU (rank = device): the same pair-slot /
receive-slot buffers are exchanged with ONE NCCL all-to-all-v per round (one
message per peer), over NVLink/NVSwitch.
"""

from __future__ import annotations

import atexit
import weakref

from paper_2303_13775_b200 import _lib


class LocalTransport:
    kind = "local"

    def all_reduce(self, t):
        pass  # all devices' gradients are summed by sg_sum_sgd in device order

    def to_owner(self, dsplit, l, send, recv, stride):
        _lib.call("sg_xfer_to_owner", _lib.ptr(dsplit.ws), dsplit.lay, l, _lib.ptr(send),
                  _lib.ptr(recv), int(stride), _lib.stream_ptr())

    def from_owner(self, dsplit, l, send_recv_layout, recv_pair_layout, stride):
        _lib.call("sg_xfer_from_owner", _lib.ptr(dsplit.ws), dsplit.lay, l,
                  _lib.ptr(send_recv_layout), _lib.ptr(recv_pair_layout), int(stride),
                  _lib.stream_ptr())


class NcclTransport:
    """Rank-local exchange over torch.distributed: NCCL all-to-all-v on GPUs.

    stage_on_host=True copies the payload through host memory and uses the
    process group's CPU collective (gloo); it exists so the rank-local code
    path can be exercised by several processes sharing one GPU in tests."""

    kind = "nccl"

    def __init__(self, rank, world_size, group=None, stage_on_host=False):
        self.rank = int(rank)
        self.world = int(world_size)
        self.group = group
        self.stage = bool(stage_on_host)

    def _a2a(self, out, inp, out_splits, in_splits):
        import torch.distributed as dist
        if not self.stage:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
            return
        o = out.cpu()
        dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
        out.copy_(o)

    def all_reduce(self, t):
        """Sum a flat gradient buffer over ranks (NCCL allreduce)."""
        import torch.distributed as dist
        if not self.stage:
            dist.all_reduce(t, group=self.group)
            return
        c = t.cpu()
        dist.all_reduce(c, group=self.group)
        t.copy_(c)

    def _splits(self, meta, l):
        r, g = self.rank, self.world
        send_rows = [int(meta.cnt[l][r][o]) for o in range(g)]
        recv_rows = [int(meta.cnt[l][s][r]) for s in range(g)]
        return send_rows, recv_rows

    def to_owner(self, dsplit, l, send, recv, stride):
        m = dsplit.host_meta()
        r = self.rank
        send_rows, recv_rows = self._splits(m, l)
        s0, s1 = int(m.ref_off[l][r]), int(m.ref_off[l][r + 1])
        r0, r1 = int(m.recv_off[l][r]), int(m.recv_off[l][r + 1])
        self._a2a(recv[r0:r1].reshape(-1), send[s0:s1].reshape(-1),
                  [c * stride for c in recv_rows], [c * stride for c in send_rows])

    def from_owner(self, dsplit, l, send_recv_layout, recv_pair_layout, stride):
        m = dsplit.host_meta()
        r = self.rank
        send_rows, recv_rows = self._splits(m, l)   # reversed roles
        s0, s1 = int(m.recv_off[l][r]), int(m.recv_off[l][r + 1])
        r0, r1 = int(m.ref_off[l][r]), int(m.ref_off[l][r + 1])
        self._a2a(recv_pair_layout[r0:r1].reshape(-1), send_recv_layout[s0:s1].reshape(-1),
                  [c * stride for c in send_rows], [c * stride for c in recv_rows])


_LIVE = weakref.WeakSet()


@atexit.register
def _close_live_transports():
    for tp in list(_LIVE):
        try:
            tp.close()
        except Exception:
            pass


class PeerTransport:
    """One rank per GPU, exchanges over peer memory (csrc/peer.cu): every
    round's buffer of every rank is mapped into its peers with CUDA IPC
    (torch's storage sharing), rows move with one kernel writing (push-to-
    owner) or reading (push-from-owner) the peers' buffers at the GLOBAL slot
    numbering every rank knows from the replicated split, and device flags
    tagged with a per-step epoch order the rounds. No sizes go to the host, so
    the rank-local step is capturable as one CUDA graph
    (engine.RankCapturedStep). The gradient all-reduce + SGD runs over the same
    mapped memory (all_reduce_sgd) and doubles as the step barrier.

    Buffers are requested per round with `shared(rows, stride)` in the same
    order on every rank (the engine's program order); the first request of a
    round allocates and exchanges handles (a collective over `group`)."""

    kind = "peer"

    def __init__(self, rank, world_size, group=None, device=None):
        import torch
        self.rank = int(rank)
        self.world = int(world_size)
        self.group = group
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        lib = _lib.load()
        self.rounds = int(lib.sg_peer_rounds())
        self._keep = []
        nflag = self.rounds * 16
        self.flags = torch.zeros(nflag + 64, dtype=torch.int32, device=self.dev)
        self.epoch = self.flags[nflag:nflag + 1]
        self.timeout = self.flags[nflag + 32:nflag + 33]
        self.peer_flags = self._share(self.flags)
        self._bufs = {}
        self._nbuf = 0
        self._nx = 0
        self._grad = None
        _LIVE.add(self)

    def close(self):
        """Synchronise and unmap the peers' buffers while CUDA is still up (also
        run at interpreter exit, before torch's own teardown: dropping IPC
        mappings during that teardown could crash the process on exit)."""
        import torch
        if self._keep:
            torch.cuda.synchronize(self.dev)
        self._bufs.clear()
        self._grad = None
        self._keep.clear()
        self.peer_flags = None
        _LIVE.discard(self)

    # -- CUDA IPC mapping -----------------------------------------------------
    def _share(self, t):
        """All-gather IPC handles of `t`'s storage; returns the g peer pointers
        (own entry = t itself) as an int64 array."""
        import numpy as np
        import torch
        import torch.distributed as dist
        st = t.untyped_storage()
        h = st._share_cuda_()
        off = t.data_ptr() - st.data_ptr()
        hs = [None] * self.world
        dist.all_gather_object(hs, (h, off), group=self.group)
        ptrs = []
        for r, (hr, offr) in enumerate(hs):
            if r == self.rank:
                ptrs.append(t.data_ptr())
                continue
            ps = torch.UntypedStorage._new_shared_cuda(*hr)
            self._keep.append(ps)
            ptrs.append(ps.data_ptr() + offr)
        self._keep.append(t)
        return np.asarray(ptrs, dtype=np.int64)

    # -- per-step protocol ------------------------------------------------------
    def begin_step(self):
        self._nbuf = 0
        self._nx = 0
        _lib.call("sg_peer_epoch", _lib.ptr(self.epoch), _lib.stream_ptr())

    def shared(self, rows, stride):
        """This round's exchange buffer (rows x stride fp32), mapped into every peer."""
        import torch
        k = self._nbuf
        self._nbuf += 1
        if k >= self.rounds:
            raise RuntimeError(f"more than {self.rounds} exchange rounds in one step")
        need = max(int(rows) * int(stride), 4)
        cur = self._bufs.get(k)
        if cur is None or cur[0].numel() < need:
            t = torch.empty(need, dtype=torch.float32, device=self.dev)
            cur = (t, self._share(t))
            self._bufs[k] = cur
        return cur[0][:need].view(-1, int(stride)) if rows else cur[0][:0].view(0, int(stride))

    def _round(self, buf):
        k = self._nx
        self._nx += 1
        t, peers = self._bufs[k]
        if buf.data_ptr() != t.data_ptr():
            raise RuntimeError("exchange buffer was not requested from this transport for this round")
        return k, peers

    def _signal_wait(self, k):
        st = _lib.stream_ptr()
        _lib.call("sg_peer_signal", _lib.ptr(self.peer_flags), self.rank, self.world, k, _lib.ptr(self.epoch), st)
        _lib.call("sg_peer_wait", _lib.ptr(self.flags), self.rank, self.world, k, _lib.ptr(self.epoch),
                  _lib.ptr(self.timeout), st)

    def peers_of(self, buf):
        """The g peer-mapped pointers of the round buffer `buf` (int64 array),
        for kernels that store into the owners' buffers themselves."""
        for t, peers in self._bufs.values():
            if t.data_ptr() == buf.data_ptr():
                return peers
        raise RuntimeError("buffer was not requested from this transport")

    def to_owner(self, dsplit, l, send, recv, stride, pushed=False):
        """Push this rank's pair-slot rows into the owners' receive buffers
        (pushed=True: the producing kernel already stored them there)."""
        k, peers = self._round(recv)
        if not pushed:
            _lib.call("sg_peer_exchange", _lib.ptr(dsplit.ws), dsplit.lay, l, self.rank, 1, _lib.ptr(send),
                      int(stride), _lib.ptr(peers), _lib.stream_ptr())
        self._signal_wait(k)

    def from_owner(self, dsplit, l, send_recv_layout, recv_pair_layout, stride):
        """Owners packed their rows (receive-slot layout) into this round's
        shared buffer; after the round's flags, pull this rank's pair slots."""
        k, peers = self._round(send_recv_layout)
        self._signal_wait(k)
        _lib.call("sg_peer_exchange", _lib.ptr(dsplit.ws), dsplit.lay, l, self.rank, 0,
                  _lib.ptr(recv_pair_layout), int(stride), _lib.ptr(peers), _lib.stream_ptr())

    def all_reduce_sgd(self, gbuf, n, params_flat, scale, grads_out=None, lr=None, num_targets=None):
        """Sum the ranks' flat gradients (+ loss slot) in rank order and apply
        the SGD step, over peer memory (the step barrier). num_targets (device
        int64 scalar) + lr: scale = lr / num_targets computed on the device."""
        import torch
        n1 = int(gbuf.numel())
        stride = (n1 + 63) // 64 * 64
        if self._grad is None or self._grad[2] != stride:
            t = torch.zeros(2 * stride, dtype=torch.float32, device=self.dev)
            self._grad = (t, self._share(t), stride)
        t, peers, stride = self._grad
        st = _lib.stream_ptr()
        _lib.call("sg_peer_grad_stage", _lib.ptr(gbuf), _lib.ptr(t), n1, stride, _lib.ptr(self.epoch), st)
        self._signal_wait(self.rounds - 1)
        if num_targets is not None:
            _lib.call("sg_peer_allreduce_sgd_nt", _lib.ptr(peers), self.world, int(n), n1, stride,
                      _lib.ptr(self.epoch), _lib.ptr(params_flat), _lib.ptr(grads_out), float(lr),
                      num_targets.data_ptr(), st)
            return
        _lib.call("sg_peer_allreduce_sgd", _lib.ptr(peers), self.world, int(n), n1, stride, _lib.ptr(self.epoch),
                  _lib.ptr(params_flat), _lib.ptr(grads_out), float(scale), st)

    def check(self):
        """Raise if a peer wait timed out (a peer process is gone)."""
        if int(self.timeout.item()):
            raise RuntimeError("peer transport: a peer never signalled (timed out)")


# ---- C5 microbenchmark -----------------------------------------------------------------

def uniform_exchange_sample(rows, g):
    """A one-layer sample whose split plan is a uniform all-to-all: device o
    owns `rows` destinations, each with an in-edge from one source vertex of
    every other device, so every (holder, owner) pair holds exactly `rows`
    reference rows (pair_count = rows * g * (g - 1)). Returns (sample, pm)."""
    import numpy as np

    from paper_2303_13775_b200.partition import PartitionMap
    from paper_2303_13775_b200.sampling import MiniBatchSample
    nt = g * rows
    asn = np.concatenate([np.repeat(np.arange(g), rows), np.arange(g)]).astype(np.int64)
    pm = PartitionMap(asn, g, float(g))
    tgt = np.arange(nt, dtype=np.int64)
    V0 = np.arange(nt + g, dtype=np.int64)
    own = tgt // rows
    # per destination: self edge, then one edge from every foreign device's source
    srcs = np.broadcast_to(np.arange(g, dtype=np.int64), (nt, g))
    keep = srcs != own[:, None]
    cross = (nt + srcs[keep]).reshape(nt, g - 1)
    src = np.concatenate([tgt[:, None], cross], axis=1).reshape(-1)
    dst = np.repeat(tgt, g)
    return MiniBatchSample(1, [V0, tgt], [(src, dst)], dst_grouped=True), pm


def exchange_microbench(rows, width, world=1, rank=0, device=None, parts=8, steps=20, warmup=3, transport=None):
    """Time the split's push-to-owner round on a uniform plan (rows per peer,
    `width` fp32 per row) through the repo's transport: LocalTransport (all
    `parts` devices on this GPU, sg_xfer_to_owner) at world = 1, the
    PeerTransport (peer stores + signal/wait) at world > 1. Returns
    {"ms": per round, "bytes": bytes sent per GPU (world > 1) or read + written
    (world = 1)}."""
    import torch

    from paper_2303_13775_b200.scheduler import DeviceSplit
    g = world if world > 1 else parts
    dev = torch.device(device) if device is not None else torch.device("cuda")
    smp, pm = uniform_exchange_sample(rows, g)
    ds = DeviceSplit.from_sample(smp, pm, None, dev)
    P = ds.pair_bound(1)
    stride = (width + 3) // 4 * 4
    if world == 1:
        tp = LocalTransport()
        send = torch.rand(P, stride, device=dev)
        recv = torch.empty(P, stride, device=dev)

        def one():
            tp.to_owner(ds, 1, send, recv, stride)
        nbytes = 2 * rows * g * (g - 1) * stride * 4
    else:
        tp = transport if transport is not None else PeerTransport(rank, world, device=dev)
        send = torch.rand(P, stride, device=dev)

        def one():
            tp.begin_step()
            recv = tp.shared(P, stride)
            tp.to_owner(ds, 1, send, recv, stride)
        nbytes = rows * (g - 1) * stride * 4
    for _ in range(warmup):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        tp.check()
    return {"ms": e0.elapsed_time(e1) / steps, "bytes": nbytes, "pairs": int(ds.pair_count(1))}
