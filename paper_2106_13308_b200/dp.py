"""Data-parallel host logic of the B200 step: which reference workers a rank
plays, how the per-rank results combine, and the one collective per step.

The reference runs L worker threads in one process (proj/src/trainer.cpp:111-306): worker w
draws from make_stream(seed, w + 1), computes its gradient with its own in-batch baseline,
and worker 0 forms the fixed-order tree mean (trainer.cpp:324-335).  Here every GPU rank
plays `workers_per_rank` consecutive workers (segments of one device batch) and the device
step all-reduces (NCCL, sum) the live gradient; Adam divides by the global worker count.
Pooled statistics are formed from exact integer cut sums.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _capi as K


@dataclass(frozen=True)
class RankPlan:
    rank: int
    world: int
    workers_per_rank: int

    @property
    def total_workers(self) -> int:
        return self.world * self.workers_per_rank

    @property
    def first_worker(self) -> int:
        return self.rank * self.workers_per_rank

    @property
    def stream0(self) -> int:
        """Stream of this rank's first worker: worker w uses make_stream(seed, w + 1)."""
        return self.first_worker + 1

    def streams(self):
        return [self.stream0 + s for s in range(self.workers_per_rank)]

    @property
    def grad_scale(self) -> float:
        """allreduce_mean's division (trainer.cpp:334), applied after the sum."""
        return 1.0 / self.total_workers


def pooled_stats(num_edges: int, n_samples: int, cut_sum: int, cut_sq_sum: int):
    """energy_and_variance over the pooled L*mbs local energies (trainer.cpp:246-248) from
    exact integer sums of cut and cut^2 (l = (|E| - 2 cut) / 4)."""
    m, v = C.c_double(), C.c_double()
    K.check(K.lib.vqmc_pooled_stats(num_edges, n_samples, cut_sum, cut_sq_sum, C.byref(m), C.byref(v)))
    return m.value, v.value


def allreduce_sums(values, group=None):
    """Sum integer statistics over ranks with torch.distributed (any backend; int64 exact)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.int64)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [int(x) for x in t.tolist()]


def share_unique_id(uid: bytes, group=None) -> bytes:
    """Broadcast rank 0's NCCL unique id (vqmc_gpu_comm_unique_id) to every rank."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return uid
    obj = [uid]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


@dataclass(frozen=True)
class Communicator:
    """What api.train(cfg, comm) needs to put this rank's handle on the step's NCCL communicator:
    the rank, the world size and rank 0's NCCL unique id (128 bytes)."""
    rank: int
    world: int
    unique_id: bytes


def make_communicator(rank: int, world: int, group=None) -> Communicator:
    """Rank 0 draws the NCCL unique id (vqmc_gpu_comm_unique_id); torch.distributed (any backend,
    already initialised) broadcasts it.  One process per GPU, as in bench.py."""
    uid = b""
    if rank == 0:
        buf = (C.c_uint8 * 128)()
        K.check(K.lib.vqmc_gpu_comm_unique_id(buf))
        uid = bytes(buf)
    uid = share_unique_id(uid, group)
    if len(uid) != 128:
        raise RuntimeError("NCCL unique id was not shared (is torch.distributed initialised?)")
    return Communicator(rank, world, uid)


def stat_limbs_decode(limbs) -> int:
    """Inverse of the step's exact-integer encoding inside the fp32 gradient all-reduce: an
    integer statistic travels as 16-bit limbs, each an exactly representable fp32 value whose
    sum over <= 256 ranks stays below 2^24 (exact); value = sum_k limb_k * 2^(16 k)."""
    v = 0
    for k, x in enumerate(limbs):
        v += int(round(float(x))) << (16 * k)
    return v


def stat_limbs_encode(value: int, count: int):
    if value < 0:
        raise ValueError("non-negative statistics only")
    out = [float((value >> (16 * k)) & 0xFFFF) for k in range(count)]
    if value >> (16 * count):
        raise ValueError("statistic does not fit the limbs")
    return out
