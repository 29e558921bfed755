"""Multi-GPU driver (torchrun flavour): edge lightcones sharded over the GPUs of
one node, one process per GPU.

Lightcones are independent (the reference already runs them on a thread pool,
proj/src/engine.cpp:531-541), so the only exchange is one reduction of the
per-edge <ZZ> terms.  Each rank plans and contracts its shard on its own GPU;
the terms vector (2m float64, zero outside the shard) is reduced to rank 0
with a single NCCL reduce (sum), and rank 0 forms
<C> = m/2 - 1/2 sum_e Re e_jk in edge order, exactly as energy_expectation
does (engine.cpp:549-560).  Summing a slot with zeros is exact, so the
N-GPU energy is bit-identical to the 1-GPU one.

Sharding is LPT (longest processing time first) on the predicted device work
of every lightcone (qtng_edge_work: complex products + adds of the reference
loop).  The fused device program is bound by FP64 issue and latency, not by
HBM bytes, so work -- not bytes -- predicts device time.  `shards_for` uses
the library's own placement (qtng_shard_edges), the one the single-process
C driver qtng_energy_multi uses, so both drivers shard identically.
"""
from __future__ import annotations

import heapq
from typing import List, Optional, Sequence

import numpy as np


def lpt_shard(costs: Sequence[float], world: int) -> List[List[int]]:
    """Greedy LPT: edges by decreasing cost onto the least-loaded rank.
    Returns each rank's edge indices in ascending order (deterministic)."""
    world = max(1, int(world))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    out: List[List[int]] = [[] for _ in range(world)]
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(s) for s in out]


def shards_for(q, g, p: int, world: int, merged: bool = False) -> List[List[int]]:
    """Each rank's edges (ascending) under the library's LPT placement."""
    own = q.shard_edges(g, p, world, merged=merged)
    return [sorted(int(i) for i in np.nonzero(own == r)[0]) for r in range(max(1, world))]


def shard_imbalance(costs: Sequence[float], shards: List[List[int]]) -> float:
    """max shard load / mean shard load (1.0 = perfect)."""
    loads = [sum(float(costs[i]) for i in s) for s in shards]
    mean = sum(loads) / max(1, len(loads))
    return max(loads) / mean if mean > 0 else 1.0


def scatter_terms(m: int, shard: Sequence[int], terms: np.ndarray) -> np.ndarray:
    """This rank's complex terms placed into a zero (2m,) float64 vector."""
    full = np.zeros(2 * m, dtype=np.float64)
    idx = np.asarray(shard, dtype=np.int64)
    full[2 * idx] = np.real(terms)
    full[2 * idx + 1] = np.imag(terms)
    return full


def energy_from_terms(m: int, full: np.ndarray) -> float:
    """<C> = m/2 - 1/2 sum Re e_jk, summed in edge order (engine.cpp:549-560)."""
    s = 0.0
    for i in range(m):
        s += float(full[2 * i])
    return 0.5 * m - 0.5 * s


def reduce_terms(full: np.ndarray, device: Optional["object"] = None, dst: int = 0) -> np.ndarray:
    """One collective: sum-reduce the per-edge term vectors to rank `dst`."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(full)
    if device is not None:
        t = t.to(device)
    dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()
