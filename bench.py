"""Benchmark of the hot path: one Picasso conflict-graph build = one step.

Metric (BASELINE.json): candidate pairs/sec in the conflict-graph build.  A step builds the
iteration-1 conflict graph of the N=1 workload — BASELINE config 2: 100,000 random Pauli
strings on 32 qubits (generate.py's generator, seed 0), PaletteParams(12.5, 2.0, seed 0):
P = 12,500 colors, L = 23 — i.e. n(n-1)/2 = 4,999,950,000 candidate pairs per step.

  value   device-resident: inputs (packed words, active ids, color lists) already in HBM;
          each step = the whole build on the device (input prep incl. color buckets and
          bucket commute masks, commuting-pair sweep, conflict-row count, compaction, fill);
          the CSR stays in HBM.  CUDA events on the builder's own stream, one pair per step;
          a 512 MiB L2-flush write runs between steps, outside the timed region.
  e2e     the public API (paper_2401_06713_b200.build) with host numpy inputs in pinned
          memory and int64 numpy outputs: H2D of the step's inputs, build, D2H of the CSR
          (members, offsets, neighbors) inside the timed region.

`--impl reference` times the reference algorithm on the host CPU instead (the C port in
oracle/, all host threads, a bounded row sample of the same workload); it never touches the
GPU.  Multi-GPU (torchrun): the pair space is sharded by rank (see distributed.py); value =
all ranks' pairs / max-over-ranks device time.
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


def make_inputs(name: str, pinned: bool = False):
    import paper_2401_06713_b200 as b200

    n, q, gseed, pct, alpha, seed = WORKLOADS[name]
    strings = b200.random_pauli_strings(n, q, seed=gseed)
    ps = b200.PauliSet.from_strings(strings)
    view = b200.pauli_view(ps)
    plan = b200.plan_iteration(1, n, b200.PaletteParams(pct, alpha, seed=seed))
    lists = b200.assign_random_lists(plan, view.active, seed)
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


def measured_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the committed
    ncu --set full capture of this bench command (profiles/roofline_traffic.json, written by
    tools/profile_summary.py); None when no capture is committed."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            rec = json.load(f).get(kernel)
        return None if rec is None else (float(rec["dram_bytes_per_launch"]), "profiles/" + rec["source"])
    except (OSError, ValueError, KeyError):
        return None


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def cpu_baseline(view, lists, seconds: float = 12.0) -> dict:
    """The reference algorithm on host cores: oracle/ C port (predicate + dense palette-mask
    intersection per pair, conflict.py:72-78), all host threads, bounded row sample."""
    from oracle.oracle import OracleInstance

    inst = OracleInstance(view.backing.words, view.active, lists, threads=1)
    n = inst.n
    threads = os.cpu_count() or 1
    rs = np.random.default_rng(0)
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
    return {"value": state["pairs"] / dt, "unit": "pairs/s", "cores": threads, "kind": "port",
            "sample": f"{state['rows']} random upper-triangle rows ({state['pairs']} pairs) of the "
                      f"same workload in {dt:.1f} s; oracle/conflict_oracle.c scan_rows "
                      "(commute predicate + palette bitmask AND per pair), one row per task"}


def bench_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    view, lists, plan = make_inputs(args.workload)
    n = view.n_active
    per_step = []
    base = None
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(view, lists, seconds=args.ref_seconds)
        if k >= args.warmup:
            per_step.append(cb["value"])
            base = cb
    value = statistics.mean(per_step)
    pairs = n * (n - 1) // 2
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * pairs / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {n} random Pauli strings x {WORKLOADS[args.workload][1]} qubits, "
                               f"P={plan.palette_size}, L={plan.list_size}, iteration-1 build",
                   "pairs_per_step": pairs, "host_cores": os.cpu_count()},
        "cpu_baseline": {**base, "value": value},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def l2_flush(buf):
    buf.fill_(1)


def bench_gpu(args) -> None:
    import torch

    import paper_2401_06713_b200 as b200
    from paper_2401_06713_b200 import _native
    from paper_2401_06713_b200.conflict import stage

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # PICASSO_FORCE_SHARDED=1 runs the sharded (torchrun) path with one rank: a one-GPU check
    # of the N>1 code path
    if world > 1 or os.environ.get("PICASSO_FORCE_SHARDED") == "1":
        from paper_2401_06713_b200 import distributed as dist_mod

        dist_mod.bench_sharded(args)
        return

    view, lists, plan = make_inputs(args.workload, pinned=True)
    n = view.n_active
    pairs = n * (n - 1) // 2
    ctx = _native.context(local)
    ctx.profiling(True)
    stage(view, lists, ctx)  # H2D of the inputs: not part of `value`
    ctx.option("k1_async", 1)  # K1 (view_edges_scanned only) next to the conflict-row passes
    stream = torch.cuda.ExternalStream(ctx.stream_handle())
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    # ---- device-resident value
    launches = 0
    for _ in range(args.warmup):
        ctx.build_device()
    times, ktimes = [], []
    torch.cuda.synchronize()
    with ClockSampler(None if args.no_clocks else local) as clocks:
        for _ in range(args.steps):
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
    ms = statistics.mean(times)
    value = pairs / (ms * 1e-3)
    edges = int(c.deg_sum) // 2
    members = int(c.members_in_range)
    kt = np.mean(np.array(ktimes), axis=0)  # [K1, K2 count, K2 fill, compaction, prep]

    # ---- end to end through the public API (pinned host inputs, numpy outputs)
    ctx.profiling(False)  # the public build runs without the per-phase events
    e2e_t = []
    for k in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gc = b200.build(view, lists)
        torch.cuda.synchronize()
        if k >= args.warmup:
            e2e_t.append(time.perf_counter() - t0)
        # bytes that crossed PCIe device -> host: members, offsets, and the neighbor ids as
        # byte gaps + exceptions (decoded into the 8-byte int64 output on the host)
        d2h = _native.context(local).last_copy_bytes()
        out_bytes = gc.members.nbytes + gc.graph.offsets.nbytes + gc.graph.neighbors.nbytes
        gc = None  # a user drops each step's graph; the next build reuses its host pages
    h2d = view.backing.words.nbytes + view.active.nbytes + lists.array.nbytes
    e2e_value = pairs / statistics.mean(e2e_t)
    e2e_steps_ms = [round(t * 1e3, 2) for t in e2e_t]

    # ---- roofline of the dominant kernel (HBM: algorithmic bytes of the conflict-row fill)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    fill_ms = float(kt[2])
    words_b = n * view.backing.words.shape[1] * 8
    # device CSR ids are int32 (widened to the API's int64 on the host during the D2H copy)
    fill_bytes = (2 * edges) * 4 + (members + 1) * 8 + members * 8 + n * plan.list_size * 4 + words_b
    achieved = fill_bytes / (fill_ms * 1e-3) / 1e9
    # the fill kernel the native layer picks for this size (abi.cu fill_rows_device)
    fill_kernel = "k_fill_blk" if n <= 131072 else "k_fill_bins"
    # the commuting-pair sweep against the survey's POPC-issue bound (1 POPC / pair / clk)
    sm_mhz = (clocks.summary().get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0))
    popc_bound = 148 * 16 * sm_mhz * 1e6
    k1_rate = pairs / (float(kt[0]) * 1e-3)

    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {n} random Pauli strings x {WORKLOADS[args.workload][1]} qubits "
                               f"(generate.py seed {WORKLOADS[args.workload][2]}), P={plan.palette_size}, "
                               f"L={plan.list_size}, iteration-1 conflict-graph build",
                   "pairs_per_step": pairs, "conflict_edges": edges,
                   "view_edges_scanned": int(c.pairs_in_shard - c.anticommuting),
                   "l2": "512 MiB flush write between timed steps",
                   "parallelism": "single GPU"},
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "ms_per_step": 1e3 * statistics.mean(e2e_t),
                "step_ms": e2e_steps_ms,
                "host_output_bytes_per_step": int(out_bytes),
                "host_output": "int64 numpy (members, offsets, neighbors); the neighbors buffer "
                               "is reused across steps once the previous step's graph is "
                               "dropped (hostpool.py); neighbor ids cross PCIe as 8- or 16-bit "
                               "gaps and are decoded on the host"},
        "gpu_launches": int(launches),
        "kernel_ms": {"commute_sweep_k1": float(kt[0]), "conflict_rows_count_k2b": float(kt[1]),
                      "conflict_rows_fill_k2b": float(kt[2]), "compaction": float(kt[3]),
                      "prep_incl_bucket_masks_k2a": float(kt[4])},
        "roofline": {"bound": "hbm", "kernel": f"conflict-row fill ({fill_kernel})",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": (measured_traffic(fill_kernel) or (None, None))[0],
                     "traffic_source": (measured_traffic(fill_kernel) or (None, None))[1],
                     "bytes_per_launch": int(fill_bytes),
                     "note": f"{fill_kernel} is instruction-issue bound, not HBM bound (ncu: IPC "
                             "2.1-2.4 of 4, DRAM throughput ~8%; profiles/*_ncu_summary.md): the "
                             "frac is reported against HBM as the contract asks",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
        "int_roofline": {"kernel": "commuting-pair sweep (k_commute_fr2, 64-bit four-Russians tables)", "achieved": k1_rate,
                         "unit": "pairs/s", "peak": popc_bound,
                         "peak_model": "148 SMs x 16 POPC/clk x measured SM clock (1 POPC per pair)",
                         "frac": k1_rate / popc_bound},
        "clocks": clocks.summary(),
    }
    if not args.no_run:
        # the whole Picasso run on this workload (GPU builds + GPU palette lists + native
        # host list coloring): end-to-end coloring time and #colors (BASELINE.json metric)
        t0 = time.perf_counter()
        res = b200.run(view, b200.PaletteParams(*WORKLOADS[args.workload][3:6]))
        line["run"] = {"seconds": time.perf_counter() - t0, "colors": res.total_colors,
                       "iterations": len(res.iterations), "oracle_edges": res.oracle_edges,
                       "peak_conflict_edges": res.peak_conflict_edges}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(view, lists, seconds=args.cpu_seconds)
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="skip the nvidia-smi sampler")
    ap.add_argument("--no-run", action="store_true", help="skip the whole-run report")
    args = ap.parse_args()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_gpu(args)


if __name__ == "__main__":
    main()
