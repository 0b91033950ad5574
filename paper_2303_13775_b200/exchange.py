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

    def to_owner(self, dsplit, l, send, recv, stride):
        _lib.call("sg_xfer_to_owner", _lib.ptr(dsplit.ws), dsplit.lay, l, _lib.ptr(send),
                  _lib.ptr(recv), int(stride), _lib.stream_ptr())

    def from_owner(self, dsplit, l, send_recv_layout, recv_pair_layout, stride):
        _lib.call("sg_xfer_from_owner", _lib.ptr(dsplit.ws), dsplit.lay, l,
                  _lib.ptr(send_recv_layout), _lib.ptr(recv_pair_layout), int(stride),
                  _lib.stream_ptr())


class NcclTransport:
    """Rank-local exchange over torch.distributed (NCCL on GPUs; gloo works
    for CPU tests of the descriptor logic)."""

    kind = "nccl"

    def __init__(self, rank, world_size, group=None):
        self.rank = int(rank)
        self.world = int(world_size)
        self.group = group

    def _splits(self, meta, l):
        r, g = self.rank, self.world
        send_rows = [int(meta.cnt[l][r][o]) for o in range(g)]
        recv_rows = [int(meta.cnt[l][s][r]) for s in range(g)]
        return send_rows, recv_rows

    def to_owner(self, dsplit, l, send, recv, stride):
        import torch.distributed as dist
        m = dsplit.host_meta()
        r = self.rank
        send_rows, recv_rows = self._splits(m, l)
        s0, s1 = int(m.ref_off[l][r]), int(m.ref_off[l][r + 1])
        r0, r1 = int(m.recv_off[l][r]), int(m.recv_off[l][r + 1])
        dist.all_to_all_single(recv[r0:r1].reshape(-1), send[s0:s1].reshape(-1),
                               [c * stride for c in recv_rows], [c * stride for c in send_rows],
                               group=self.group)

    def from_owner(self, dsplit, l, send_recv_layout, recv_pair_layout, stride):
        import torch.distributed as dist
        m = dsplit.host_meta()
        r = self.rank
        send_rows, recv_rows = self._splits(m, l)   # reversed roles
        s0, s1 = int(m.recv_off[l][r]), int(m.recv_off[l][r + 1])
        r0, r1 = int(m.ref_off[l][r]), int(m.ref_off[l][r + 1])
        dist.all_to_all_single(recv_pair_layout[r0:r1].reshape(-1),
                               send_recv_layout[s0:s1].reshape(-1),
                               [c * stride for c in send_rows], [c * stride for c in recv_rows],
                               group=self.group)
