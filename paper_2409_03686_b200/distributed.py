"""Row sharding of the exit-measure matrix across GPUs.

Rows of A (poles) are independent, and every walk's RNG stream is keyed by
its GLOBAL pole id, so any partition of the rows reproduces the single-GPU
counts exactly.  Poles go to ranks cyclically (pole i -> rank i mod N), which
balances pole-dependent walk lengths (SURVEY hard part 9).  The one exchange
step is an all-gather of the int64 count rows and step statistics over
torch.distributed -- NCCL over NVLink/NVSwitch on the GPU box, gloo in the CPU
tests.  One process per GPU.
"""

from __future__ import annotations

import numpy as np

from .backend import AccumulateResult, Plan, pack_geometry
from .errors import WalkBudgetError


def shard_rows(n_poles: int, world: int, rank: int) -> np.ndarray:
    """Global pole ids owned by ``rank`` (cyclic)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return np.arange(rank, n_poles, world, dtype=np.int64)


def gather_rows(local, n_poles: int, world: int, group=None):
    """All-gather per-rank row blocks (shard order from shard_rows) into the
    full (n_poles, ...) tensor on every rank.  ``local`` is a torch tensor
    whose first dimension is this rank's shard length."""
    import torch
    import torch.distributed as dist

    m_pad = -(-n_poles // world)
    pad = torch.zeros((m_pad,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = torch.empty((n_poles,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    for r in range(world):
        ids = torch.as_tensor(shard_rows(n_poles, world, r), device=local.device)
        out[ids] = parts[r][: ids.numel()]
    return out


def cyclic_gather_index(n_poles: int, world: int, m_pad: int, device=None):
    """Row index into the rank-major all-gather of per-rank blocks of m_pad
    rows: global pole g lives in rank g % world's block at row g // world."""
    import torch

    g = torch.arange(n_poles, device=device)
    return (g % world) * m_pad + g // world


def exchange_rows(buf, gathered, index, m_pad: int, row: int, out, group=None) -> None:
    """The one exchange of a strong-scaling step: ONE all-gather of every
    rank's flat block (count rows (m_pad, row) first), then the un-permute of
    the gathered rows into pole order (``out``, (n_poles, row)) on the
    device.  ``gathered`` is (world, len(buf)), ``index`` from
    cyclic_gather_index."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "gloo" and buf.is_cuda:  # host exchange (harness test)
        g = gathered.cpu()
        dist.all_gather_into_tensor(g.view(-1), buf.cpu(), group=group)
        gathered.copy_(g)
    else:
        dist.all_gather_into_tensor(gathered.view(-1), buf, group=group)
    rows = gathered[:, : m_pad * row].reshape(gathered.shape[0] * m_pad, row)
    torch.index_select(rows, 0, index, out=out)


_NO_ERROR = np.iinfo(np.int64).max


def agree_on_budget_error(err, n_rep: int, max_steps: int, device, group=None) -> None:
    """Collective: every rank contributes its first budget overrun (or none);
    the lexicographically smallest GLOBAL (pole, replicate) over all ranks is
    raised as WalkBudgetError on EVERY rank, before any data exchange -- so
    no rank leaves the collective sequence while the others block in the
    gather (S/backend.py:189-192: the first failing job in job order)."""
    import torch
    import torch.distributed as dist

    key = _NO_ERROR if err is None else int(err.pole) * int(n_rep) + int(err.replicate)
    t = torch.tensor([key], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    k = int(t.item())
    if k != _NO_ERROR:
        raise WalkBudgetError(k // int(n_rep), k % int(n_rep), max_steps)


def run_accumulate_sharded(dom, ksqrt, poles, seed: int, eps: float, max_steps: int,
                           n_rep: int, side0, side1, *, precision: str | None = None,
                           chain: str | None = None, group=None) -> AccumulateResult:
    """run_accumulate over all ranks of the default (or given) process group:
    each rank walks its cyclic row shard on its own GPU (LOCAL_RANK), budget
    errors are agreed on collectively, the rows are all-gathered, and every
    rank returns the full result.  IDW families (REF64) gather their
    fractional float64 rows instead of the int64 counts."""
    import os

    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = int(os.environ.get("EXITMEASURE_B200_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    poles = np.ascontiguousarray(poles, dtype=np.float64)
    n_poles = poles.shape[0]
    ids = shard_rows(n_poles, world, rank)
    geom = pack_geometry(dom)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", device) if nccl else torch.device("cpu")
    err = None
    counts = raw = stats = None
    ms = 0.0
    with Plan(geom, ksqrt, poles[ids], eps, max_steps, side0, side1, precision, chain, device,
              pole_ids=ids) as plan:
        try:
            if plan.idw:  # fractional rows: the REF64 raw path, float64 exchange
                res = plan.run_raw(seed, n_rep)
                raw = torch.as_tensor(np.concatenate([res.raw0, res.raw1], 1), device=dev)
                stats = torch.as_tensor(np.stack([res.steps_sum, res.steps_sq_sum,
                                                  res.steps_max], 1), device=dev)
            elif nccl:  # rows stay in HBM: walk, all-gather over NVLink, one copy back
                row = plan.n0 + plan.n1
                counts = torch.zeros((len(ids), row), dtype=torch.int64, device=dev)
                stats3 = torch.zeros((3, len(ids)), dtype=torch.int64, device=dev)
                plan.run_device(seed, n_rep, counts.data_ptr(), stats3.data_ptr(),
                                torch.cuda.current_stream(dev).cuda_stream)
                torch.cuda.current_stream(dev).synchronize()
                plan.check()
                stats = stats3.t().contiguous()
                ms = plan.last_stats()[0]
            else:
                res = plan.run(seed, n_rep)
                counts = torch.as_tensor(res.counts)
                stats = torch.as_tensor(np.stack([res.steps_sum, res.steps_sq_sum,
                                                  res.steps_max], 1))
                ms = res.kernel_ms
        except WalkBudgetError as e:  # global pole id (plan pole_ids)
            err = e
    agree_on_budget_error(err, n_rep, max_steps, dev, group)
    full_stats = gather_rows(stats, n_poles, world, group).cpu().numpy()
    n0 = int(side0.size)
    if raw is not None:
        full_raw = gather_rows(raw, n_poles, world, group).cpu().numpy()
        return AccumulateResult(full_raw[:, :n0].copy(), full_raw[:, n0:].copy(),
                                full_stats[:, 0].copy(), full_stats[:, 1].copy(),
                                full_stats[:, 2].copy(), 0, None, ms, n0=n0)
    full_counts = gather_rows(counts, n_poles, world, group).cpu().numpy()
    return AccumulateResult(None, None, full_stats[:, 0].copy(), full_stats[:, 1].copy(),
                            full_stats[:, 2].copy(), 0, full_counts, ms, n0=n0)
