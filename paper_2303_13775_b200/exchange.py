"""Transports for the push-to-owner / push-from-owner rounds.

LocalTransport: all g devices live in this process (one GPU): one copy kernel
per round moves every holder->owner block (the reference's in-process
exchange, engine.py:125-156, without the Python loops).

NcclTransport: one process per GPU (rank = device): the same pair-slot /
receive-slot buffers are exchanged with ONE NCCL all-to-all-v per round (one
message per peer), over NVLink/NVSwitch.
"""

from __future__ import annotations

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
