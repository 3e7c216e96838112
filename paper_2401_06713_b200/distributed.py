"""Pair-space sharding of the conflict build across GPUs (one process per GPU).

SURVEY.md §8(e).  Every rank holds the (small, replicated) inputs and runs:

  1. the input prep (encode, color buckets) — replicated, O(n L) — and the owned bucket
     masks (K2a) for the member rows in its own row range only (options own_rows_lo/hi:
     the commute-mask rows, the bulk of K2a, divide by the world size);
  2. the commuting-pair sweep over its share of the upper triangle (K1 work items
     rank/world) and the conflict-row count over its contiguous row range (K2c);
  3. all-reduce of the four totals and all-gather of the per-row degrees (4 B per row);
  4. the budget check (identical on every rank — the same exception everywhere);
  5. the fill of its own rows (K2f) into a device slice (int32 ids);
  6. a gather of the slices, in rank order, to the root rank (default), which widens them
     and copies the canonical int64 CSR to its host once; ``gather="all"`` all-gathers
     instead (every rank returns the whole graph).

Rows are independent (each GPU generates full rows from the color buckets), so the only
exchanges are the degree all-gather and the slice gather.  With ``backend="nccl"`` both run
on device tensors over NVLink; with gloo (CPU tests) they run on host tensors.  The per-rank
compute goes through an *engine* (the CUDA context by default; tests substitute an
oracle-backed engine to check this host logic without a GPU).

``run_sharded`` is the whole Picasso run on N GPUs (driver.py:272-385, the reference's
Algorithm 1): every rank takes part in each sharded build, the root colors the conflict
graph on the host (the list coloring is sequential in its draws) and broadcasts the outcome,
so every rank ends with the identical coloring — the single-GPU run's and the reference's.
"""

from __future__ import annotations

import os
from typing import Optional

import numpy as np

from . import _native, hostpool
from .conflict import _error_types, _lists_as_csr, _result_types, one_phase_projection


def row_ranges(n: int, world: int) -> list:
    """Contiguous, near-equal row ranges [r0, r1) per rank."""
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


class NativeEngine:
    """Per-rank compute on this rank's GPU through the C ABI."""

    def __init__(self, device: Optional[int] = None):
        self.ctx = _native.context(device)

    def set_inputs(self, words, num_qubits, active, data, off, L, base, P, rows=None):
        # the owned-mask rows this rank's count and fill will read (the prep runs here)
        lo, hi = rows if rows is not None else (0, -1)
        self.ctx.option("own_rows_lo", lo)
        self.ctx.option("own_rows_hi", hi)
        try:
            self.ctx.set_inputs(words, num_qubits, active, data, off, L, base, P)
        finally:
            self.ctx.option("own_rows_lo", 0)
            self.ctx.option("own_rows_hi", -1)

    def count(self, shard, nshards, r0, r1):
        c = self.ctx.count(shard, nshards, r0, r1)
        return dict(anticommuting=int(c.anticommuting), pairs=int(c.pairs_in_shard),
                    deg_sum=int(c.deg_sum), members=int(c.members_in_range))

    def degrees(self, rows):
        return self.ctx.degrees(rows)

    def fill_rows_device(self, global_deg, out_ptr, out32: bool = False, absolute: bool = False):
        """The rank's CSR slice into a device buffer, int64 or int32 (None: bounds only);
        ``absolute``: out_ptr is the whole CSR's base (the rows go to their global offsets)."""
        import torch

        g = torch.from_numpy(np.ascontiguousarray(global_deg, dtype=np.int32)).cuda()
        mx = int(global_deg.max()) if global_deg.size else 0
        torch.cuda.synchronize()  # the upload (torch's stream) before the context's stream reads it
        self.ctx.option("rows_out32", 1 if out32 else 0)
        self.ctx.option("rows_out_abs", 1 if absolute else 0)
        try:
            lohi = self.ctx.fill_rows_device(g.data_ptr(), mx, out_ptr)
        finally:
            self.ctx.option("rows_out32", 0)
            self.ctx.option("rows_out_abs", 0)
        torch.cuda.synchronize()
        return lohi

    # peer-memory exchange (exchange="p2p"): the root's exported buffer, mapped by every rank
    def exchange_buffer(self, nbytes: int):
        return self.ctx.exchange_buffer(nbytes)

    def exchange_map(self, handle: bytes) -> int:
        return self.ctx.exchange_map(handle)

    def ids_to_host(self, ptr: int, out: np.ndarray) -> None:
        self.ctx.ids_to_host(ptr, out)

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


def _share_handle(dist, handle: Optional[bytes], root: int, dev) -> bytes:
    """The root's 64-byte IPC handle on every rank (a broadcast over the process group)."""
    import torch

    t = torch.zeros(64, dtype=torch.uint8)
    if handle is not None:
        t[:] = torch.frombuffer(bytearray(handle), dtype=torch.uint8)
    t = t.to(dev)
    dist.broadcast(t, src=root)
    return bytes(t.cpu().numpy().tobytes())


def p2p_available(engine) -> bool:
    return hasattr(engine, "exchange_buffer") and hasattr(engine, "fill_rows_device")


def build_sharded(view, lists, *, edge_budget: Optional[int] = None, threads: int = 1,
                  block_pairs: int = 1 << 20, two_phase: bool = True, engine=None,
                  gather: str = "root", root: int = 0, exchange: str = "auto"):
    """The conflict build of ``conflict.build``, sharded over the default process group.

    ``gather="root"``: the root rank returns the canonical ConflictGraph (bit-identical to
    the single-GPU build and to the reference); the other ranks return its header — the
    same members, offsets, edge_count and view_edges_scanned, with an empty neighbor array.
    ``gather="all"``: every rank returns the whole graph.  Budget errors are raised on every
    rank, with the caller's exception class (conflict._error_types).

    ``exchange`` (gather="root"): "p2p" — the root exports one device buffer for the CSR's
    int32 ids (a CUDA IPC handle, broadcast over the process group) and every rank's fill
    stores its rows straight into it over NVLink while it produces them; "collective" — each
    rank fills a local slice and the process group gathers the slices to the root; "auto"
    (default) — p2p when the engine is the native (GPU) one.
    """
    import torch
    import torch.distributed as dist

    if gather not in ("root", "all"):
        raise ValueError("gather must be 'root' or 'all'")
    if exchange not in ("auto", "p2p", "collective"):
        raise ValueError("exchange must be 'auto', 'p2p' or 'collective'")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = _coll_device(dist)
    engine = engine or NativeEngine()
    CG, EG = _result_types(view)
    budget_error, _ = _error_types(view)
    words = np.ascontiguousarray(view.backing.words, dtype=np.uint64)
    active = np.ascontiguousarray(view.active, dtype=np.int64)
    n = int(active.size)
    data, off, L = _lists_as_csr(lists, n)
    ranges = row_ranges(n, world)
    r0, r1 = ranges[rank]
    engine.set_inputs(words, int(view.backing.num_qubits), active, data, off, L,
                      int(lists.palette_base), int(lists.palette_size), rows=(r0, r1))
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
            raise budget_error(total, edge_budget)
        gdegu = _all_gather_rows(dist, degu_local.astype(np.int32), ranges, dev)
        raise budget_error(one_phase_projection(gdegu, block_pairs, edge_budget), edge_budget)
    has = gdeg > 0
    members_ids = active[has]
    offsets = np.zeros(int(has.sum()) + 1, dtype=np.int64)
    np.cumsum(gdeg[has].astype(np.int64), out=offsets[1:])
    assert members_ids.size == members and offsets[-1] == 2 * total
    # every slice's length follows from the gathered degrees
    starts = np.concatenate([[0], np.cumsum(gdeg.astype(np.int64))])
    lens_np = [int(starts[b] - starts[a]) for a, b in ranges]
    p2p = gather == "root" and (exchange == "p2p" or (exchange == "auto" and p2p_available(engine)))
    if p2p:
        if not p2p_available(engine):
            raise ValueError("exchange='p2p' needs the native (GPU) engine")
        # the root's CSR buffer in its HBM; every rank's fill writes its rows into it
        ptr, handle = engine.exchange_buffer(4 * max(2 * total, 1)) if rank == root else (0, None)
        handle = _share_handle(dist, handle, root, dev)
        base = ptr if rank == root else engine.exchange_map(handle)
        if lens_np[rank]:
            engine.fill_rows_device(gdeg, base, out32=True, absolute=True)
        dist.barrier()  # every rank's fill has completed (its stream synchronized)
        if rank == root:
            nbr = hostpool.empty_int64(2 * total)
            engine.ids_to_host(ptr, nbr)
        else:
            nbr = np.zeros(0, dtype=np.int64)
        return CG(members=members_ids, graph=EG(n=int(members_ids.size), offsets=offsets,
                                                  neighbors=nbr),
                  edge_count=total, view_edges_scanned=pairs - anti)
    width = max(max(lens_np, default=0), 1)
    device_fill = dev.type == "cuda" and hasattr(engine, "fill_rows_device")
    t = torch.zeros(width, dtype=torch.int32 if device_fill else torch.int64, device=dev)
    if device_fill:  # NCCL: the slice is filled into a device buffer, never crosses PCIe
        if lens_np[rank]:
            engine.fill_rows_device(gdeg, t.data_ptr(), out32=True)
    else:
        lo, hi, vals = engine.fill_rows(gdeg, True)
        assert hi - lo == lens_np[rank]
        if hi > lo:
            t[: hi - lo] = torch.from_numpy(vals).to(dev)
    receive = gather == "all" or rank == root
    if gather == "all":
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
    else:
        parts = [torch.empty_like(t) for _ in range(world)] if rank == root else None
        dist.gather(t, parts, dst=root)
    if not receive:
        nbr = np.zeros(0, dtype=np.int64)
    elif device_fill:
        # widen on the device, then one copy per slice into the pooled (pinned) host buffer
        # the single-GPU build also reuses
        nbr = hostpool.empty_int64(2 * total)
        host = torch.from_numpy(nbr)
        pos = 0
        for r in range(world):
            if lens_np[r]:
                host[pos:pos + lens_np[r]].copy_(parts[r][: lens_np[r]].to(torch.int64))
                pos += lens_np[r]
    else:
        nbr = np.concatenate([p[: lens_np[r]].cpu().numpy() for r, p in enumerate(parts)]) \
            if world else np.zeros(0, np.int64)
    if receive:
        assert nbr.size == 2 * total
    return CG(members=members_ids, graph=EG(n=int(members_ids.size), offsets=offsets, neighbors=nbr),
              edge_count=total, view_edges_scanned=pairs - anti)


def run_sharded(view, params, *, strategy: str = "dynamic", edge_budget: Optional[int] = None,
                block_pairs: int = 1 << 20, engine=None, root: int = 0, exchange: str = "auto"):
    """The whole Picasso run (driver.run) with every conflict build sharded over the default
    process group.  The root rank colors each conflict graph (list_coloring, the reference's
    draw order) and broadcasts the outcome; every rank returns the identical ColoringResult."""
    import torch.distributed as dist

    from . import driver, list_coloring
    from .list_coloring import ConflictColoringOutcome

    rank = dist.get_rank()

    def builder(v, lists, **kw):
        kw.pop("threads", None)
        return build_sharded(v, lists, engine=engine, gather="root", root=root,
                             exchange=exchange, **kw)

    def coloring(gc, lists, strategy, seed, iteration, view=None):
        box = [None]
        if rank == root:
            o = list_coloring.color_conflict_graph(gc, lists, strategy=strategy, seed=seed,
                                                   iteration=iteration, view=view)
            ids = np.fromiter(o.colored.keys(), dtype=np.int64, count=len(o.colored))
            cols = np.fromiter(o.colored.values(), dtype=np.int64, count=len(o.colored))
            box[0] = (ids, cols, o.uncolored, o.colors_used, o.empties, o.removal_ops)
        dist.broadcast_object_list(box, src=root)
        ids, cols, unc, used, empties, removals = box[0]
        return ConflictColoringOutcome(colored=dict(zip(ids.tolist(), cols.tolist())),
                                       uncolored=unc, colors_used=used, empties=empties,
                                       removal_ops=removals)

    return driver.run(view, params, strategy=strategy, edge_budget=edge_budget,
                      block_pairs=block_pairs, builder=builder, conflict_coloring=coloring)


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
    ranges = row_ranges(n, world)
    r0, r1 = ranges[rank]
    # the prep computes the owned-mask rows of this rank's row range only, and launches this
    # rank's K1 shard on a side stream once the buckets are sorted (beside the owned masks,
    # the count and the fill; joined at the end of the step)
    ctx.option("own_rows_lo", r0)
    ctx.option("own_rows_hi", r1)
    ctx.option("k1_async", 1)
    ctx.option("k1_early", 1)
    ctx.option("k1_shard", rank)
    ctx.option("k1_nshards", world)
    stage(view, lists, ctx)
    width = max(b - a for a, b in ranges)
    ctx.option("rows_out32", 1)  # the timed step exchanges int32 slices
    deg_local = torch.zeros(width, dtype=torch.int32, device=dev)
    gdeg_parts = torch.zeros(world * width, dtype=torch.int32, device=dev)
    # exchange: "p2p" (default) — every rank's fill stores its rows into the root's CSR
    # buffer over NVLink (CUDA IPC mapping, set up once: the buffer is reused every step);
    # "collective" (PICASSO_EXCHANGE=collective) — int32 slices gathered by NCCL
    exchange = os.environ.get("PICASSO_EXCHANGE", "p2p")
    xbase = [0]
    if exchange == "p2p":
        ctx.option("rows_out_abs", 1)
        ctx.prep_device()
        ctx.count(rank, world, r0, r1)
        ctx.k1_result()
        ctx.degrees_device(deg_local.data_ptr())
        dist.all_gather_into_tensor(gdeg_parts, deg_local)
        total_ids = int(gdeg_parts.to(torch.int64).sum().item())
        ptr, handle = ctx.exchange_buffer(4 * max(total_ids, 1)) if rank == 0 else (0, None)
        handle = _share_handle(dist, handle, 0, dev)
        xbase[0] = ptr if rank == 0 else ctx.exchange_map(handle)

    def step():
        # input prep (buckets replicated, owned masks of this rank's rows) + count of its shard
        ctx.prep_device()
        c = ctx.count(rank, world, r0, r1)
        ctx.degrees_device(deg_local.data_ptr())
        dist.all_gather_into_tensor(gdeg_parts, deg_local)
        gdeg = torch.cat([gdeg_parts[k * width: k * width + (ranges[k][1] - ranges[k][0])]
                          for k in range(world)])
        mx = int(gdeg.max().item()) if n else 0
        if exchange == "p2p":  # the rows go straight into the root's HBM
            ctx.fill_rows_device(gdeg.data_ptr(), mx, xbase[0])
            ctx.k1_result()  # this rank's K1 shard has finished too
            dist.barrier()
            return c
        lo, hi = ctx.fill_rows_device(gdeg.data_ptr(), mx, None)
        lens = torch.tensor([hi - lo], dtype=torch.int64, device=dev)
        all_lens = torch.zeros(world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(all_lens, lens)
        w = int(all_lens.max().item())
        buf = torch.zeros(max(w, 1), dtype=torch.int32, device=dev)  # int32 ids: half the exchange
        ctx.fill_rows_device(gdeg.data_ptr(), mx, buf.data_ptr())
        # the slices gathered to the root rank's HBM, in rank order (the canonical CSR)
        parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, parts, dst=0)
        ctx.k1_result()
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
    ctx.option("rows_out_abs", 0)
    for k, v in (("k1_async", 0), ("k1_early", 2), ("k1_shard", 0), ("k1_nshards", 1)):
        ctx.option(k, v)
    ctx.option("own_rows_lo", 0)
    ctx.option("own_rows_hi", -1)
    # ---- end to end through the public sharded build (host inputs in, the canonical int64
    # CSR on the root rank's host out), max over ranks
    import time

    e2e = []
    nnz = 0
    for k in range(1 + args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        gc = build_sharded(view, lists, gather="root")
        torch.cuda.synchronize()
        if k >= 1:
            e2e.append(time.perf_counter() - t0)
        nnz = int(gc.graph.neighbors.size)
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
            "data": "synthetic", "config": bench_mod.config_for(args.workload, world),
            "sharding": "K1 work items and K2 row ranges by rank, owned masks of the rank's "
                        "rows, NCCL degree all-gather; " + (
                            "each rank's fill stores its int32 CSR rows straight into rank 0's "
                            "buffer over NVLink (CUDA IPC peer memory)" if exchange == "p2p" else
                            "int32 CSR slices gathered to rank 0 by NCCL"),
            "e2e": {"value": pairs / e2e_s, "unit": "pairs/s",
                    # root rank: its inputs and the gathered degrees up; down: the degrees and
                    # the canonical int64 CSR (members and offsets are derived on the host
                    # from the degrees)
                    "h2d_bytes_per_step": int(h2d + 4 * n),
                    "d2h_bytes_per_step": int(8 * nnz + 4 * n),
                    "ms_per_step": 1e3 * e2e_s,
                    "api": "distributed.build_sharded (gather='root': rank 0 returns the "
                           "canonical CSR)"},
            "gpu_launches": int(launches.item()),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
