"""Multi-GPU evaluation: contiguous observation shards, one small all-reduce.

Observations are independent given the (replicated) dataset, and their
contributions combine by summation (reference: engine/__init__.py:155-170), so
rank r evaluates rows [i0_r, i1_r) -- the same (i0, i1) range the reference
runners take (_kernels.pyx:392-393) -- and one SUM all-reduce of L+1 doubles
(the totals and a failure count) finishes the evaluation.  Only when the count
is non-zero does a second, MAX all-reduce recover the lowest failing index.
One process per GPU; ``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

from .errors import NotPositiveDefinite


def shard_bounds(n: int, world_size: int, rank: int) -> tuple:
    """Contiguous, near-equal split of [0, n): the first n % world ranks get one extra row."""
    if not 0 <= rank < world_size:
        raise ValueError("rank outside [0, world_size)")
    base, extra = divmod(n, world_size)
    i0 = rank * base + min(rank, extra)
    return i0, i0 + base + (1 if rank < extra else 0)


_PINNED: dict = {}


def combine_partials(vec, group=None):
    """All-reduce one rank's (L+2,) result tensor in place and return (totals, first_fail).

    vec[0:L] totals, vec[L] failure count, vec[L+1] = -(lowest failing index)-1 or -inf
    (layout of vb200_eval_async).  Works on CUDA tensors (NCCL) and CPU tensors (gloo).
    """
    import torch
    import torch.distributed as dist

    L = vec.shape[0] - 2
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    if multi:
        dist.all_reduce(vec[:L + 1], op=dist.ReduceOp.SUM, group=group)
    # ONE device-to-host copy (and one synchronisation) per evaluation; the branch on the summed failure
    # count is taken on the host, identically on every rank
    if vec.is_cuda:  # pinned staging buffer + one stream synchronisation (a pageable .to("cpu") costs ~20 us more)
        key = (vec.device.index, vec.shape[0])
        stage = _PINNED.get(key)
        if stage is None:
            stage = _PINNED[key] = torch.empty(vec.shape[0], dtype=torch.float64).pin_memory()
        stage.copy_(vec.detach(), non_blocking=True)
        torch.cuda.current_stream(vec.device).synchronize()
        host = stage.numpy().copy()
    else:
        host = vec.detach().to(torch.float64).numpy().copy()
    if multi and host[L] > 0.0:  # rare: somebody failed -- recover the lowest failing index
        dist.all_reduce(vec[L + 1:], op=dist.ReduceOp.MAX, group=group)
        host[L + 1] = float(vec[L + 1])
    first_fail = -1
    if host[L] > 0.0:
        first_fail = int(round(-host[L + 1] - 1.0))
    return host[:L].copy(), first_fail


class ShardedEvaluator:
    """Callable theta -> ProfiledEvaluation over all ranks' shards (drives ``inference.fit``).

    Every rank builds a ``DeviceProblem`` for its own rows and calls the evaluator
    with the same theta; all ranks get the same assembled result, so they take the
    same Fisher-scoring decisions without a broadcast.
    """

    def __init__(self, ds, nn, family: str, jitter: float = 0.0, group=None, device=None, layout: str = "auto"):
        import torch.distributed as dist

        from .engine import DeviceProblem

        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group, self.jitter, self.family = group, float(jitter), family
        self.n, self.p = ds.n, ds.p
        self.i0, self.i1 = shard_bounds(ds.n, self.world, self.rank)
        self.problem = DeviceProblem(ds, nn, family, device=device, row0=self.i0, rows=self.i1 - self.i0,
                                     layout=layout)

    def totals(self, theta) -> np.ndarray:
        vec = self.problem.totals_async(theta, self.jitter)
        totals, first = combine_partials(vec, self.group)
        if first >= 0:
            # the pivot is known on the rank that owns the failing row; an evaluation issued chunk by chunk behind
            # the upload latches only its last piece's failure word, so ask the plain (single-launch) path
            piv = -1
            if self.i0 <= first < self.i1:
                try:
                    self.problem.totals(theta, self.jitter)
                except NotPositiveDefinite as err:
                    piv = err.pivot if err.observation == first else -1
            raise NotPositiveDefinite(pivot=piv, observation=first)
        return totals

    def __call__(self, theta):
        from .engine import parts_from_flat
        from .inference import assemble

        theta = np.asarray(theta, dtype=np.float64)
        return assemble(parts_from_flat(self.totals(theta), self.p, theta.shape[0]), self.n)

    def close(self):
        self.problem.close()
