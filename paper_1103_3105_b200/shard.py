"""Multi-GPU bulk step: one sharded gputx handle per GPU, records moved by all-to-all.

The engine (include/gputx.h "Sharding") packs, merges and executes; this module only
moves the packed device buffers between shards:
  C1  records per (source, destination) pair          all_to_all of the count vector
  C2  cross-shard transactions [ts, type, len, params] all_to_all of u32 words
  C3  remote fragment outputs [ts, out words]          all_to_all of u32 words
With backend "nccl" the buffers stay in HBM and move over NVLink; "gloo" (CPU tests)
moves host tensors.  `LocalShards` runs G shards of one process on one GPU with the
same exchange done by device copies (parity tests on a single GPU).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .gputx import Database


def all_to_all_records(send: torch.Tensor, counts: list[int], stride: int, group=None):
    """Exchange fixed-stride u32 records: `send` holds sum(counts) records grouped by
    destination rank.  Returns (recv tensor, records received)."""
    world = dist.get_world_size(group)
    dev = send.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    c_send = torch.tensor(counts, dtype=torch.int64, device=dev)
    c_recv = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(c_recv, c_send, group=group)                       # C1
    rc = [int(x) for x in c_recv.tolist()]
    total = sum(rc)
    payload = send[:sum(counts) * stride].to(dev)
    recv = torch.empty(max(total, 1) * stride, dtype=torch.int32, device=dev)
    dist.all_to_all_single(recv[:total * stride], payload, [c * stride for c in rc],
                           [c * stride for c in counts], group=group)          # C2 / C3
    if recv.device != send.device:
        recv = recv.to(send.device)
    if recv.is_cuda:
        # the engine reads recv on its own stream: the exchange's writes (NCCL, or the
        # host-to-device copy after gloo) must have landed first (include/gputx.h)
        torch.cuda.current_stream(recv.device).synchronize()
    return recv, total


def connect_p2p(db: Database, group=None):
    """Map every rank's exchange arena into this rank (CUDA IPC over NVLink / NVSwitch):
    the blobs are all-gathered once with torch.distributed (host plumbing only); from then
    on records move by the library's own kernels (gputx_shard_dispatch / return)."""
    blobs = [None] * dist.get_world_size(group)
    dist.all_gather_object(blobs, db.shard_export(), group=group)
    db.shard_connect(blobs)
    db.p2p = True


def step(db: Database, home, strategy: str, group=None, on_device: bool = False) -> dict:
    """One bulk on this rank's shard.  Connected (connect_p2p): dispatch over peer memory,
    receive, execute, return, collect -- no host staging, no collective.  Otherwise: pack,
    all-to-all with torch.distributed, submit, execute, return, merge.
    `home` = this rank's home transactions with global ts (numpy or device tensors)."""
    if getattr(db, "p2p", False):
        db.shard_dispatch(home, on_device=on_device)
        db.shard_receive()
        st = db.execute(strategy)
        db.shard_return()
        db.shard_collect()
        return st
    send, counts = db.shard_pack(home, on_device=on_device)
    recv, n = all_to_all_records(send, counts, db.shard_stride(False), group)
    db.shard_submit(recv, n)
    st = db.execute(strategy)
    rsend, rcounts = db.shard_return_pack()
    rrecv, rn = all_to_all_records(rsend, rcounts, db.shard_stride(True), group)
    db.shard_return_merge(rrecv, rn)
    return st


class LocalShards:
    """G shard handles in one process on one GPU; the all-to-all is a device gather, or
    (p2p=True) the library's fused peer-memory exchange between the handles."""

    def __init__(self, dbs: list[Database], p2p: bool = False):
        self.dbs = dbs
        self.p2p = p2p
        if p2p:
            Database.shard_connect_local(dbs)

    @staticmethod
    def _exchange(sends, counts, stride):
        G = len(sends)
        recvs = []
        for q in range(G):
            parts = []
            for r in range(G):
                off = sum(counts[r][:q])
                parts.append(sends[r][off * stride:(off + counts[r][q]) * stride])
            n = sum(counts[r][q] for r in range(G))
            recvs.append((torch.cat(parts) if n else sends[q][:stride].clone(), n))
        return recvs

    def step(self, homes, strategy: str, on_device: bool = False) -> list[dict]:
        dbs = self.dbs
        if self.p2p:              # every dispatch before any receive (receive waits for all peers)
            for db, h in zip(dbs, homes):
                db.shard_dispatch(h, on_device=on_device)
            for db in dbs:
                db.shard_receive()
            stats = [db.execute(strategy) for db in dbs]
            for db in dbs:
                db.shard_return()
            for db in dbs:
                db.shard_collect()
            return stats
        packed = [db.shard_pack(h, on_device=on_device) for db, h in zip(dbs, homes)]
        recvs = self._exchange([p[0] for p in packed], [p[1] for p in packed], dbs[0].shard_stride(False))
        torch.cuda.current_stream().synchronize()          # the device gathers have landed
        for db, (rv, n) in zip(dbs, recvs):
            db.shard_submit(rv, n)
        stats = [db.execute(strategy) for db in dbs]
        rp = [db.shard_return_pack() for db in dbs]
        rr = self._exchange([p[0] for p in rp], [p[1] for p in rp], dbs[0].shard_stride(True))
        torch.cuda.current_stream().synchronize()
        for db, (rv, n) in zip(dbs, rr):
            db.shard_return_merge(rv, n)
        return stats
