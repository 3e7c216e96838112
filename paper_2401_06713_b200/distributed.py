"""Pair-space sharding of the conflict build across GPUs (one process per GPU).

SURVEY.md §8(e).  Every rank holds the (small, replicated) inputs and runs:

  1. the commuting-pair sweep over its share of the upper triangle (K1 tile shard
     rank/world) and the conflict-row count over its contiguous row range (K2);
  2. all-reduce of the four totals and all-gather of the per-row degrees (n int32);
  3. the budget check (identical on every rank — same exception everywhere);
  4. the fill of its own rows, written straight into its slice of the global CSR (global
     offsets and compact ids come from the gathered degrees);
  5. all-gather of the slices, in rank order, into the canonical CSR.

Rows are independent (each GPU generates full rows from the color buckets), so the only
exchanges are the degree all-gather (4 bytes per row) and the CSR slice all-gather.  With
``backend="nccl"`` both run on device tensors over NVLink; with gloo (CPU tests) they run on
host tensors.  The per-rank compute goes through an *engine* (the CUDA context by default;
tests substitute an oracle-backed engine to check this host logic without a GPU).
"""

from __future__ import annotations

import os
from typing import Optional

import numpy as np

from . import _native, hostpool
from .conflict import ConflictGraph, _lists_as_csr, _result_types, one_phase_projection
from .errors import EdgeBudgetExceededError


def row_ranges(n: int, world: int) -> list:
    """Contiguous, near-equal row ranges [r0, r1) per rank."""
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


class NativeEngine:
    """Per-rank compute on this rank's GPU through the C ABI."""

    def __init__(self, device: Optional[int] = None):
        self.ctx = _native.context(device)

    def set_inputs(self, words, num_qubits, active, data, off, L, base, P):
        self.ctx.set_inputs(words, num_qubits, active, data, off, L, base, P)

    def count(self, shard, nshards, r0, r1):
        c = self.ctx.count(shard, nshards, r0, r1)
        return dict(anticommuting=int(c.anticommuting), pairs=int(c.pairs_in_shard),
                    deg_sum=int(c.deg_sum), members=int(c.members_in_range))

    def degrees(self, rows):
        return self.ctx.degrees(rows)

    def fill_rows_device(self, global_deg, out_ptr, out32: bool = False):
        """The rank's CSR slice into a device buffer, int64 or int32 (None: bounds only)."""
        import torch

        g = torch.from_numpy(np.ascontiguousarray(global_deg, dtype=np.int32)).cuda()
        mx = int(global_deg.max()) if global_deg.size else 0
        torch.cuda.synchronize()  # the upload (torch's stream) before the context's stream reads it
        self.ctx.option("rows_out32", 1 if out32 else 0)
        try:
            lohi = self.ctx.fill_rows_device(g.data_ptr(), mx, out_ptr)
        finally:
            self.ctx.option("rows_out32", 0)
        torch.cuda.synchronize()
        return lohi

    def fill_rows(self, global_deg, want_values: bool):
        lo, hi = self.ctx.fill_rows(global_deg, None)
        if not want_values:
            return lo, hi, None
        out = np.empty(hi - lo, dtype=np.int64)
        if hi > lo:
            self.ctx.fill_rows(global_deg, out)
        return lo, hi, out


def _coll_device(dist):
    import torch

    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
        else torch.device("cpu")


def _all_gather_rows(dist, local: np.ndarray, ranges, dev) -> np.ndarray:
    """Gather variable-length int arrays (one per rank, in rank order) on every rank."""
    import torch

    world = len(ranges)
    sizes = [r1 - r0 for r0, r1 in ranges]
    width = max(sizes) if sizes else 0
    t = torch.zeros(width, dtype=torch.int64 if local.dtype == np.int64 else torch.int32, device=dev)
    if local.size:
        t[: local.size] = torch.from_numpy(np.ascontiguousarray(local)).to(dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return np.concatenate([o[: sizes[r]].cpu().numpy() for r, o in enumerate(out)]) if world else local


def build_sharded(view, lists, *, edge_budget: Optional[int] = None, threads: int = 1,
                  block_pairs: int = 1 << 20, two_phase: bool = True, engine=None):
    """The conflict build of ``conflict.build``, sharded over the default process group.

    Every rank returns the same canonical ConflictGraph (bit-identical to the single-GPU
    build and to the reference).
    """
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    dev = _coll_device(dist)
    engine = engine or NativeEngine()
    CG, EG = _result_types(view)
    words = np.ascontiguousarray(view.backing.words, dtype=np.uint64)
    active = np.ascontiguousarray(view.active, dtype=np.int64)
    n = int(active.size)
    data, off, L = _lists_as_csr(lists, n)
    engine.set_inputs(words, int(view.backing.num_qubits), active, data, off, L,
                      int(lists.palette_base), int(lists.palette_size))
    ranges = row_ranges(n, world)
    r0, r1 = ranges[rank]
    c = engine.count(rank, world, r0, r1)
    tot = torch.tensor([c["anticommuting"], c["pairs"], c["deg_sum"], c["members"]],
                       dtype=torch.int64, device=dev)
    dist.all_reduce(tot)
    anti, pairs, deg_sum, members = (int(x) for x in tot.cpu().tolist())
    deg_local, degu_local = engine.degrees(r1 - r0)
    gdeg = _all_gather_rows(dist, deg_local.astype(np.int32), ranges, dev)
    total = deg_sum // 2
    if edge_budget is not None and total > edge_budget:
        if two_phase:
            raise EdgeBudgetExceededError(total, edge_budget)
        gdegu = _all_gather_rows(dist, degu_local.astype(np.int32), ranges, dev)
        raise EdgeBudgetExceededError(one_phase_projection(gdegu, block_pairs, edge_budget),
                                      edge_budget)
    device_fill = dev.type == "cuda" and hasattr(engine, "fill_rows_device")
    if device_fill:  # NCCL: the slice is filled into a device buffer, never crosses PCIe
        lo, hi = engine.fill_rows_device(gdeg, None)
    else:
        lo, hi, slice_vals = engine.fill_rows(gdeg, True)
    # slices are contiguous in rank order; gather their lengths first
    lens = torch.tensor([hi - lo], dtype=torch.int64, device=dev)
    all_lens = [torch.empty_like(lens) for _ in range(world)]
    dist.all_gather(all_lens, lens)
    lens_np = [int(x.item()) for x in all_lens]
    width = max(lens_np) if lens_np else 0
    t = torch.zeros(max(width, 1), dtype=torch.int32 if device_fill else torch.int64, device=dev)
    if device_fill:
        if hi > lo:
            engine.fill_rows_device(gdeg, t.data_ptr(), out32=True)
    elif hi > lo:
        t[: hi - lo] = torch.from_numpy(slice_vals).to(dev)
    total_len = sum(lens_np)
    if device_fill:
        # all-gather the int32 slices over NVLink, widen on the device, then one DMA of the
        # canonical CSR into the pooled (pinned) host buffer the single-GPU build also reuses
        out = torch.empty(world * max(width, 1), dtype=torch.int32, device=dev)
        dist.all_gather_into_tensor(out, t)
        nbr = hostpool.empty_int64(total_len)
        pos = 0
        host = torch.from_numpy(nbr)
        for r in range(world):
            if lens_np[r]:
                seg = out[r * max(width, 1): r * max(width, 1) + lens_np[r]].to(torch.int64)
                host[pos:pos + lens_np[r]].copy_(seg)
                pos += lens_np[r]
    else:
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        nbr = np.concatenate([p[: lens_np[r]].cpu().numpy() for r, p in enumerate(parts)]) \
            if world else np.zeros(0, np.int64)
    has = gdeg > 0
    members_ids = active[has]
    offsets = np.zeros(int(has.sum()) + 1, dtype=np.int64)
    np.cumsum(gdeg[has].astype(np.int64), out=offsets[1:])
    assert offsets[-1] == nbr.size == 2 * total
    assert members_ids.size == members
    return CG(members=members_ids, graph=EG(n=int(members_ids.size), offsets=offsets, neighbors=nbr),
              edge_count=total, view_edges_scanned=pairs - anti)


def bench_sharded(args) -> None:
    """bench.py under torchrun: device-resident sharded builds, NCCL merge, max over ranks."""
    import json
    import statistics

    import torch
    import torch.distributed as dist

    import bench as bench_mod
    from .conflict import stage

    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    view, lists, plan = bench_mod.make_inputs(args.workload)
    n = view.n_active
    pairs = n * (n - 1) // 2
    ctx = _native.context(local)
    stage(view, lists, ctx)
    ranges = row_ranges(n, world)
    r0, r1 = ranges[rank]
    width = max(b - a for a, b in ranges)
    ctx.option("rows_out32", 1)  # the timed step exchanges int32 slices
    deg_local = torch.zeros(width, dtype=torch.int32, device=dev)
    gdeg_parts = torch.zeros(world * width, dtype=torch.int32, device=dev)

    def step():
        # input prep (replicated on every rank) + count of this rank's shard
        ctx.prep_device()
        c = ctx.count(rank, world, r0, r1)
        ctx.degrees_device(deg_local.data_ptr())
        dist.all_gather_into_tensor(gdeg_parts, deg_local)
        gdeg = torch.cat([gdeg_parts[k * width: k * width + (ranges[k][1] - ranges[k][0])]
                          for k in range(world)])
        mx = int(gdeg.max().item()) if n else 0
        lo, hi = ctx.fill_rows_device(gdeg.data_ptr(), mx, None)
        lens = torch.tensor([hi - lo], dtype=torch.int64, device=dev)
        all_lens = torch.zeros(world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(all_lens, lens)
        w = int(all_lens.max().item())
        buf = torch.zeros(max(w, 1), dtype=torch.int32, device=dev)  # int32 ids: half the exchange
        ctx.fill_rows_device(gdeg.data_ptr(), mx, buf.data_ptr())
        out = torch.empty(world * max(w, 1), dtype=torch.int32, device=dev)
        dist.all_gather_into_tensor(out, buf)
        return c

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    times = []
    l0 = ctx.launch_total()
    with bench_mod.ClockSampler(None if args.no_clocks else local) as clocks:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = torch.tensor([ctx.launch_total() - l0], dtype=torch.int64, device=dev)
    dist.all_reduce(launches)
    t = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    ctx.option("rows_out32", 0)
    # ---- end to end through the public sharded build (host inputs in, the canonical int64
    # CSR on every rank out), max over ranks
    import time

    e2e = []
    for k in range(1 + args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        gc = build_sharded(view, lists)
        torch.cuda.synchronize()
        if k >= 1:
            e2e.append(time.perf_counter() - t0)
        nnz = int(gc.graph.neighbors.size)
        members = int(gc.members.size)
        gc = None
    te = torch.tensor([statistics.mean(e2e)], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    h2d = view.backing.words.nbytes + view.active.nbytes + lists.array.nbytes
    if rank == 0:
        line = {
            "metric": bench_mod.METRIC, "value": pairs / (ms * 1e-3), "unit": "pairs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": f"{args.workload}: n={n}, P={plan.palette_size}, L={plan.list_size}",
                       "pairs_per_step": pairs,
                       "parallelism": f"pair-space shards x{world} (K1 tiles + K2 row ranges), "
                                      "NCCL degree all-gather + int32 CSR slice all-gather",
                       "l2": "inputs replicated per rank; no flush (the CSR slices exceed L2)"},
            "e2e": {"value": pairs / e2e_s, "unit": "pairs/s",
                    # per rank: its inputs and the gathered degrees up; down: the degrees and
                    # the canonical int64 CSR (every rank returns the whole graph; members and
                    # offsets are derived on the host from the degrees)
                    "h2d_bytes_per_step": int(h2d + 4 * n),
                    "d2h_bytes_per_step": int(8 * nnz + 4 * n),
                    "ms_per_step": 1e3 * e2e_s,
                    "api": "distributed.build_sharded (every rank returns the canonical CSR)"},
            "gpu_launches": int(launches.item()),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
