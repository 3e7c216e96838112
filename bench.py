"""Benchmark of the hot path: one Picasso conflict-graph build = one step.

Metric (BASELINE.json): candidate pairs/sec in the conflict-graph build.  A step builds the
iteration-1 conflict graph of the N=1 workload.  The default (headline) workload is the
north-star configuration, BASELINE config 3: 1,000,000 random Pauli strings on 64 qubits
(generate.py's generator, seed 0), PaletteParams(12.5, 2.0, seed 0): P = 125,000 colors,
L = 28, i.e. n(n-1)/2 = 499,999,500,000 candidate pairs per step.  Config 2 (100k x 32q) is
reported as a secondary object inside the same line (``secondary``).

  value   device-resident: inputs (packed words, active ids, color lists) already in HBM;
          each step = the whole build on the device (input prep incl. color buckets and
          owned bucket masks, commuting-pair sweep, conflict-row count, compaction, fill);
          the CSR stays in HBM.  CUDA events on the builder's own stream, one pair per step;
          a 512 MiB L2-flush write runs between steps, outside the timed region.
  e2e     the public API (paper_2401_06713_b200.build) with host numpy inputs in pinned
          memory and int64 numpy outputs: H2D of the step's inputs, build, D2H of the CSR
          (members, offsets, neighbors) inside the timed region.

`--impl reference` times the reference algorithm on the host CPU instead (the C port of
conflict.py:72-78 in oracle/, all host threads): each step is a bounded random-row sample of
the same workload; its pairs/s counts the reference's two scans of every pair (the
two-phase build, conflict.py:110-130), so value = pairs / (2 x scan time).  It never touches
the GPU or this package's native library.  Multi-GPU (torchrun): the pair space is sharded by
rank (see distributed.py); value = all ranks' pairs / max-over-ranks device time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate pairs/sec in conflict-graph build"
WORKLOADS = {
    # name: (n, q, gen_seed, palette_pct, alpha, seed)
    "c1": (2_000, 16, 0, 12.5, 2.0, 0),
    "c2": (100_000, 32, 0, 12.5, 2.0, 0),
    "c3": (1_000_000, 64, 0, 12.5, 2.0, 0),
}


def make_inputs(name: str, pinned: bool = False, device_lists: bool = True):
    """The workload's view, iteration-1 color lists and plan.  ``device_lists=False`` draws
    the lists on the host (the reference arm must not load this package's native library);
    both draws are bit-identical (tests/test_gpu_parity.py)."""
    import paper_2401_06713_b200 as b200

    n, q, gseed, pct, alpha, seed = WORKLOADS[name]
    strings = b200.random_pauli_strings(n, q, seed=gseed)
    ps = b200.PauliSet.from_strings(strings)
    del strings
    view = b200.pauli_view(ps)
    plan = b200.plan_iteration(1, n, b200.PaletteParams(pct, alpha, seed=seed))
    lists = b200.assign_random_lists(plan, view.active, seed, device=None if device_lists else False)
    if pinned:
        import torch

        def pin(a):
            t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0].copy()).dtype, pin_memory=True)
            out = t.numpy()
            out[...] = a
            return out

        ps = b200.PauliSet(ps.strings, pin(np.asarray(ps.words)))
        view = b200.pauli_view(ps)
        lists = b200.ColorLists.from_array(view.active, pin(lists.array), lists.palette_base,
                                           lists.palette_size)
    return view, lists, plan


def config_for(name: str, world: int = 1) -> dict:
    """The ``config`` object, identical in both arms (the driver compares them)."""
    n, q, gseed, pct, alpha, seed = WORKLOADS[name]
    import math

    P = max(1, math.ceil(pct / 100.0 * n))
    L = min(P, max(1, round(alpha * math.log(n))))
    return {"workload": f"{name}: {n} random Pauli strings x {q} qubits (generate.py seed {gseed}), "
                        f"palette {pct}% (P={P}), alpha {alpha} (L={L}), seed {seed}; "
                        "iteration-1 conflict-graph build",
            "pairs_per_step": n * (n - 1) // 2,
            "l2": "512 MiB flush write between timed device steps",
            "parallelism": "single GPU" if world == 1 else f"pair-space shards x{world}"}


def host_cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in-process through NVML
    (a 50 ms polling thread; no nvidia-smi child process competing with the host thread that
    drives the GPU)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._thread = None

    def _run(self, nvml, h):
        while not self._stop.is_set():
            try:
                sm = nvml.nvmlDeviceGetClockInfo(h, nvml.NVML_CLOCK_SM)
                mx = nvml.nvmlDeviceGetMaxClockInfo(h, nvml.NVML_CLOCK_SM)
                rs = nvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), int(rs)))
            except Exception:  # noqa: BLE001 - sampling is best effort
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.device is None:
            return self
        try:
            import pynvml as nvml

            nvml.nvmlInit()
            h = nvml.nvmlDeviceGetHandleByIndex(self.device)
            self._thread = threading.Thread(target=self._run, args=(nvml, h), daemon=True)
            self._thread.start()
        except Exception:  # noqa: BLE001 - no NVML: report "unsampled"
            self._thread = None
        time.sleep(0.1)
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            time.sleep(0.1)
            self._stop.set()
            self._thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        mx = max(s[1] for s in self.samples)
        sm = [s[0] for s in self.samples]
        busy = [x for x in sm if x > 0.5 * mx] or sm
        reasons = sorted({name for _, _, r in self.samples
                          for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": reasons}


def measured_traffic(kernel: str, workload: str = ""):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` on `workload`, from
    the committed ncu --set full capture of this bench command (profiles/roofline_traffic.json,
    written by tools/profile_summary.py); None when no capture is committed."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            recs = json.load(f)
        rec = recs.get(f"{workload}:{kernel}")
        return None if rec is None else (float(rec["dram_bytes_per_launch"]), "profiles/" + rec["source"])
    except (OSError, ValueError, KeyError):
        return None


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def cpu_baseline(view, lists, seconds: float = 12.0, inst=None) -> dict:
    """The reference algorithm on host cores: oracle/ C port (predicate + dense palette-mask
    intersection per pair, conflict.py:72-78), all host threads, bounded random-row sample.
    The reference scans every pair twice (two-phase count + fill, conflict.py:110-130), so the
    build's pairs/s is half the scan rate."""
    from oracle.oracle import OracleInstance

    if inst is None:
        inst = OracleInstance(view.backing.words, view.active, lists, threads=1)
    n = inst.n
    threads = os.cpu_count() or 1
    rs = np.random.default_rng(int(time.time() * 1e6) & 0xFFFF)
    rows = rs.permutation(n - 1)  # random rows of the upper triangle
    lock = threading.Lock()
    state = {"next": 0, "pairs": 0, "rows": 0}
    deadline = time.perf_counter() + seconds

    def worker():
        while time.perf_counter() < deadline:
            with lock:
                k = state["next"]
                state["next"] += 1
            if k >= rows.size:
                return
            r = int(rows[k])
            pairs, _, _ = inst.scan_rows(r, r + 1)
            with lock:
                state["pairs"] += pairs
                state["rows"] += 1

    t0 = time.perf_counter()
    ts = [threading.Thread(target=worker) for _ in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    value = state["pairs"] / dt / 2.0
    full = n * (n - 1) // 2
    return {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
            "cpu": host_cpu_model(), "seconds": dt,
            "sample": f"{state['rows']} random upper-triangle rows ({state['pairs']} pairs) of the "
                      f"same workload scanned in {dt:.1f} s by oracle/conflict_oracle.c scan_rows "
                      "(commute predicate + dense palette-bitmask AND per pair, one row per task, "
                      "all host threads); the reference scans each pair twice (two-phase), so "
                      "value = pairs / (2 x time)",
            "extrapolated": {"full_build_s": 2 * full / (state["pairs"] / dt),
                             "how": "2 x n(n-1)/2 pairs at the sampled scan rate"}}


def bench_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.oracle import OracleInstance

    view, lists, plan = make_inputs(args.workload, device_lists=False)
    inst = OracleInstance(view.backing.words, view.active, lists, threads=1)
    per_step, step_s = [], []
    base = None
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(view, lists, seconds=args.ref_seconds, inst=inst)
        if k >= args.warmup:
            per_step.append(cb["value"])
            step_s.append(cb["seconds"])
            base = cb
    value = statistics.mean(per_step)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(step_s), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config_for(args.workload),
        "step": "a bounded sample of the build: random rows scanned for "
                f"{args.ref_seconds:.0f} s per step (ms_per_step is the sample's wall time, not "
                "a full build; the full build is extrapolated in cpu_baseline.extrapolated)",
        "cpu_baseline": {**base, "value": value},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def l2_flush(buf):
    buf.fill_(1)


def smem_peak(sm_mhz: float) -> tuple:
    """Shared-memory load peak (GB/s) for K1's lookup shape: the measured B/clk/SM of
    tools/probe/smem_bw.cu (profiles/smem_peak.json) x 148 SMs x the SM clock."""
    try:
        with open(os.path.join(ROOT, "profiles", "smem_peak.json")) as f:
            rec = json.load(f)
        bpc, src = float(rec["lds128_quarter_bytes_per_clk_per_sm"]), "profiles/smem_peak.json (measured)"
    except (OSError, ValueError, KeyError):
        bpc, src = 128.0, "nominal 128 B/clk/SM (no measured peak committed)"
    return bpc * 148 * sm_mhz * 1e6 / 1e9, src, bpc


def k1_table_bytes_per_pair(q: int) -> float:
    """Shared-memory bytes one pair costs in K1 (k_commute_fr8, K = 64*ceil(q/32) bits <= 256:
    one EB-byte table entry per 8-bit slice per 8*EB partners = K/64 bytes; k_commute_fr: one
    4-byte entry per 4-bit slice per 32 partners)."""
    K = 64 * ((q + 31) // 32)
    return K / 64.0 if K <= 256 else 4.0 * (K // 4) / 32.0


def device_steps(ctx, stream, steps: int, warmup: int, flush, clocks=None):
    """``steps`` timed device-resident builds (CUDA events on the builder's stream)."""
    import torch

    for _ in range(warmup):
        ctx.build_device()
    times, ktimes, launches = [], [], 0
    torch.cuda.synchronize()
    for _ in range(steps):
        l2_flush(flush)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c, nl = ctx.build_device()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        ktimes.append(ctx.kernel_times())
        launches += nl
    torch.cuda.synchronize()
    return c, times, np.mean(np.array(ktimes), axis=0), launches


def e2e_steps(view, lists, steps: int, warmup: int, device: int):
    """The public build from pinned host inputs to int64 numpy outputs, wall clock."""
    import torch

    import paper_2401_06713_b200 as b200
    from paper_2401_06713_b200 import _native

    t_steps, d2h, out_bytes = [], 0, 0
    for k in range(warmup + steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gc = b200.build(view, lists)
        torch.cuda.synchronize()
        if k >= warmup:
            t_steps.append(time.perf_counter() - t0)
        # bytes that crossed PCIe device -> host: members, offsets, and the neighbor ids as
        # byte gaps + exceptions (decoded into the 8-byte int64 output on the host)
        d2h = _native.context(device).last_copy_bytes()
        out_bytes = gc.members.nbytes + gc.graph.offsets.nbytes + gc.graph.neighbors.nbytes
        gc = None  # a user drops each step's graph; the next build reuses its host pages
    h2d = view.backing.words.nbytes + view.active.nbytes + lists.array.nbytes
    return t_steps, int(h2d), int(d2h), int(out_bytes)


def measure_workload(name, args, local, clocks_on: bool):
    import torch

    from paper_2401_06713_b200 import _native
    from paper_2401_06713_b200.conflict import stage

    view, lists, plan = make_inputs(name, pinned=True)
    n = view.n_active
    q = WORKLOADS[name][1]
    pairs = n * (n - 1) // 2
    ctx = _native.context(local)
    ctx.profiling(True)
    ctx.option("k1_async", 1)  # K1 (view_edges_scanned only) on a side stream, from the prep
    stage(view, lists, ctx)  # H2D of the inputs: not part of `value`
    stream = torch.cuda.ExternalStream(ctx.stream_handle())
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    with ClockSampler(local if clocks_on else None) as clocks:
        c, times, kt, launches = device_steps(ctx, stream, args.steps, args.warmup, flush)
    # K1 alone (outside the timed region): one build with K1 on the builder's stream, 16 warps,
    # nothing beside it — the kernel's own fraction of its bound, next to the in-step one
    ctx.option("k1_async", 0)
    ctx.build_device()  # (warm-up: the 16-warp K1's first launch also loads its module)
    l2_flush(flush)
    ctx.build_device()
    k1_alone_ms = float(ctx.kernel_times()[0])
    ctx.option("k1_async", 1)
    del flush
    ctx.profiling(False)  # the public build runs without the per-phase events
    e2e_t, h2d, d2h, out_bytes = e2e_steps(view, lists, args.steps, args.warmup, local)
    ms = statistics.mean(times)
    edges = int(c.deg_sum) // 2
    members = int(c.members_in_range)
    sm_mhz = clocks.summary().get("sm_mhz") or measured_peaks().get("sm_max_mhz", 1965.0)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6553.0)
    # K1 against the shared-memory bound of its table lookups
    k1_ms = float(kt[0])
    bpp = k1_table_bytes_per_pair(q)
    k1_kernel = "k_commute_fr8" if q <= 128 else "k_commute_fr"
    speak, speak_src, bpc = smem_peak(sm_mhz)
    k1_ach = pairs * bpp / (k1_ms * 1e-3) / 1e9
    k1_traffic = measured_traffic(k1_kernel, name) or (None, None)
    roof_k1 = {"bound": "smem", "kernel": f"commuting-pair sweep K1 ({k1_kernel})",
               "achieved": k1_ach, "peak": speak, "unit": "GB/s", "frac": k1_ach / speak,
               "traffic": k1_traffic[0], "traffic_source": k1_traffic[1],
               "bytes_per_launch": int(pairs * bpp), "launch_ms": k1_ms,
               "alone": {"launch_ms": k1_alone_ms,
                         "achieved": pairs * bpp / (k1_alone_ms * 1e-3) / 1e9,
                         "frac": pairs * bpp / (k1_alone_ms * 1e-3) / 1e9 / speak,
                         "note": "one build with K1 alone on the builder's stream (16 warps); "
                                 "in the timed steps K1 (8 warps) shares every SM with the "
                                 "owned-mask kernel, which finishes inside K1's launch"},
               "note": f"algorithmic bytes = shared-memory table bytes: {bpp} B per pair (one "
                       "32-byte table entry per 8-bit slice per 256 partners, read as LDS.128 by "
                       "lane pairs, 4 rows per quarter-warp on distinct bank groups) x n(n-1)/2 "
                       "pairs; K1 reads "
                       "~0 HBM (traffic), its bound is the shared-memory pipe. peak = "
                       f"{bpc:.1f} B/clk/SM x 148 x {sm_mhz:.0f} MHz ({speak_src})"}
    # the conflict-row fill against HBM (algorithmic bytes: CSR ids written + rows read)
    fill_ms = float(kt[2])
    words_b = n * view.backing.words.shape[1] * 8
    fill_bytes = (2 * edges) * 4 + (members + 1) * 8 + members * 8 + n * plan.list_size * 4 + words_b
    fill_ach = fill_bytes / (fill_ms * 1e-3) / 1e9
    fill_kernel = "k_fill_bins" if n >= 40000 else "k_fill_blk"  # the auto choice (abi.cu)
    fill_traffic = measured_traffic(fill_kernel, name) or (None, None)
    roof_fill = {"bound": "hbm", "kernel": f"conflict-row fill ({fill_kernel})", "achieved": fill_ach,
                 "peak": hbm, "unit": "GB/s", "frac": fill_ach / hbm, "traffic": fill_traffic[0],
                 "traffic_source": fill_traffic[1], "bytes_per_launch": int(fill_bytes),
                 "launch_ms": fill_ms,
                 "note": "algorithmic bytes = int32 CSR ids written + offsets/members + the rows' "
                         "lists and words read; the fill is instruction-issue bound (ncu "
                         "summaries in profiles/)",
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"}
    dominant = roof_k1 if k1_ms >= fill_ms else roof_fill
    other = roof_fill if dominant is roof_k1 else roof_k1
    out = {
        "value": pairs / (ms * 1e-3), "ms_per_step": ms, "step_ms": [round(t, 3) for t in times],
        "pairs": pairs, "edges": edges, "view_edges_scanned": int(c.pairs_in_shard - c.anticommuting),
        "launches": launches, "clocks": clocks.summary(),
        "e2e": {"value": pairs / statistics.mean(e2e_t), "unit": "pairs/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": 1e3 * statistics.mean(e2e_t),
                "step_ms": [round(t * 1e3, 2) for t in e2e_t],
                "host_output_bytes_per_step": out_bytes,
                "host_output": "int64 numpy (members, offsets, neighbors); the neighbors buffer "
                               "is reused across steps once the previous step's graph is "
                               "dropped (hostpool.py); neighbor ids cross PCIe as 8- or 16-bit "
                               "gaps and are decoded on the host"},
        "kernel_ms": {"commute_sweep_k1": float(kt[0]), "conflict_rows_count_k2c": float(kt[1]),
                      "conflict_rows_fill_k2f": float(kt[2]), "compaction": float(kt[3]),
                      "prep_incl_owned_masks_k2a": float(kt[4]),
                      "note": "K1 runs on a side stream concurrently with the prep/count/fill "
                              "chain, so the phases overlap and do not add up to ms_per_step"},
        "roofline": dominant, "roofline_other": other,
        "view": view, "lists": lists, "plan": plan,
    }
    return out


def bench_gpu(args) -> None:
    import torch

    import paper_2401_06713_b200 as b200

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # PICASSO_FORCE_SHARDED=1 runs the sharded (torchrun) path with one rank: a one-GPU check
    # of the N>1 code path
    if world > 1 or os.environ.get("PICASSO_FORCE_SHARDED") == "1":
        from paper_2401_06713_b200 import distributed as dist_mod

        dist_mod.bench_sharded(args)
        return

    m = measure_workload(args.workload, args, local, not args.no_clocks)
    line = {
        "metric": METRIC, "value": m["value"], "unit": "pairs/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_for(args.workload),
        "build": {"conflict_edges": m["edges"], "view_edges_scanned": m["view_edges_scanned"],
                  "step_ms": m["step_ms"]},
        "e2e": m["e2e"], "gpu_launches": int(m["launches"]), "kernel_ms": m["kernel_ms"],
        "roofline": m["roofline"], "roofline_other": m["roofline_other"], "clocks": m["clocks"],
    }
    view, lists = m["view"], m["lists"]
    if not args.no_run:
        # the whole Picasso run on this workload (GPU builds + GPU palette lists + native
        # host list coloring): end-to-end coloring time and #colors (BASELINE.json metric),
        # checked against the committed golden coloring (tests/golden/scale.json)
        t0 = time.perf_counter()
        res = b200.run(view, b200.PaletteParams(*WORKLOADS[args.workload][3:6]))
        run = {"seconds": time.perf_counter() - t0, "colors": res.total_colors,
               "iterations": len(res.iterations), "oracle_edges": res.oracle_edges,
               "peak_conflict_edges": res.peak_conflict_edges}
        try:
            import hashlib

            with open(os.path.join(ROOT, "tests", "golden", "scale.json")) as f:
                gold = json.load(f)["runs"][args.workload]
            sha = hashlib.sha256(np.ascontiguousarray(res.color, dtype=np.int64).data).hexdigest()[:16]
            run["golden_color_sha"] = gold["color_sha"]
            run["identical_to_golden"] = bool(sha == gold["color_sha"] and
                                              res.total_colors == gold["colors"])
        except (OSError, KeyError, ValueError):
            run["identical_to_golden"] = None
        # the same run without materializing each iteration's CSR on the host (counts-only
        # builds + the word-predicate list coloring: driver.run(conflict_rows=False))
        t0 = time.perf_counter()
        res2 = b200.run(view, b200.PaletteParams(*WORKLOADS[args.workload][3:6]), conflict_rows=False)
        import hashlib

        run["counts_only"] = {
            "seconds": time.perf_counter() - t0, "colors": res2.total_colors,
            "identical_to_full_run": bool(np.array_equal(res2.color, res.color)),
            "color_sha": hashlib.sha256(np.ascontiguousarray(res2.color, dtype=np.int64).data).hexdigest()[:16]}
        line["run"] = run
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(view, lists, seconds=args.cpu_seconds)
    del view, lists, m
    if args.secondary and args.secondary != args.workload:
        s = measure_workload(args.secondary, args, local, False)
        line["secondary"] = {"config": config_for(args.secondary), "value": s["value"],
                             "unit": "pairs/s", "ms_per_step": s["ms_per_step"],
                             "e2e": {k: s["e2e"][k] for k in ("value", "unit", "ms_per_step",
                                                            "step_ms", "h2d_bytes_per_step",
                                                            "d2h_bytes_per_step")},
                             "kernel_ms": s["kernel_ms"], "roofline": s["roofline"],
                             "roofline_other": s["roofline_other"], "gpu_launches": s["launches"]}
        line["gpu_launches"] += int(s["launches"])
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--secondary", default="c2", help="second workload reported inside the line ('' = none)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-seconds", type=float, default=5.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="skip the NVML clock sampler")
    ap.add_argument("--no-run", action="store_true", help="skip the whole-run report")
    args = ap.parse_args()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_gpu(args)


if __name__ == "__main__":
    main()
