#!/usr/bin/env python
"""Benchmark: skyline input points/s (+ dominance tests/s) on B200 vs the
reference CPU engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

A step is one complete skyline query (sky_run: partition -> representatives
-> local skylines -> merge -> ascending ids on the host) over the config's
synthetic input. Default workload: BASELINE configs[2] (correlated N=10M
d=8, grid 2^8, q=5, NoSeq) -- the largest input of the five that fits one
GPU (320 MB > L2); `--config 1..5` selects the others. A 512 MiB buffer is
written and read back between timed steps (L2 flush; the read drains the dirty lines), outside the timed region.

`value` is device-resident (inputs already in HBM); `e2e` goes through the
public API with pinned host buffers (H2D of the rows and D2H of the ids
inside the timed region). Multi-GPU: one process per GPU under torchrun;
timing is the max over ranks of CUDA-event time.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "skyline input points/sec + dominance tests/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "input points/s"
# Issue cost of one pair test on an SM (4 SMSPs; fma and alu pipes each take
# 2 cycles per warp instruction, B300_MICROARCH.md "Pipe rates"):
#  - d <= 16, packed monotone codes: 2 word subtractions (IMAD, fma pipe) +
#    1 LOP3 + 1/2 VIMNMX3 fold (alu pipe) per test -> fma pipe bound,
#    4 cycles per 32 tests per SMSP -> 32 tests/clk/SM;
#  - d > 16, FP32 coordinates: d FSETP-class compares on the alu pipe ->
#    64/d tests/clk/SM.
PACKED_TESTS_PER_CLK_PER_SM = 32
FP32_COMPARES_PER_CLK_PER_SM = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, help="BASELINE config 1..5 (default 3 = configs[2])")
    ap.add_argument("--n", type=int, default=None, help="override N (parity/debug only)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def ncu_traffic(tag):
    """DRAM bytes (read + write) per launch of the dominance kernel, mean over
    the launches of one `ncu --set full` capture committed under profiles/."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_summary.json")), reverse=True):
        try:
            with open(path) as f:
                launches = json.load(f).get(tag) or []
        except (OSError, ValueError):
            continue
        v = [e["dram_traffic_bytes"] for e in launches if "relsky3" in e.get("kernel", "")]
        if v:
            return statistics.mean(v), os.path.relpath(path, ROOT) + f" [{tag}, {len(v)} k_relsky3 launches]"
    return None, None


def ncu_pipe_mix(tag):
    """alu / fma pipe utilisation, warps active and SM clock of the dominance
    kernel (k_relsky3, duration-weighted over the launches) from the
    committed `ncu --set full` summary, or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_summary.json")), reverse=True):
        try:
            with open(path) as f:
                launches = [e for e in (json.load(f).get(tag) or []) if "relsky3" in e.get("kernel", "")]
        except (OSError, ValueError):
            continue
        if launches:
            w = sum(e.get("duration_ms", 0.0) for e in launches) or 1.0
            mix = {k: sum(e.get(k, 0.0) * e.get("duration_ms", 0.0) for e in launches) / w
                   for k in ("alu_pipe_pct", "fma_pipe_pct", "warps_active_pct", "sm_throughput_pct")}
            mix["source"] = os.path.relpath(path, ROOT) + f" [{tag}, {len(launches)} k_relsky3 launches]"
            return mix
    return None


def ncu_stream_traffic(tag):
    """DRAM bytes (read + write) per step of the HBM streaming passes from the
    committed ncu summary (`stream` entries), or (None, None)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_summary.json")), reverse=True):
        try:
            with open(path) as f:
                launches = (json.load(f).get("stream") or {}).get(tag) or []
        except (OSError, ValueError, AttributeError):
            continue
        if launches:
            return sum(e["dram_traffic_bytes"] for e in launches), os.path.relpath(path, ROOT) + f" [stream/{tag}]"
    return None, None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed
    region: NVML every 10 ms (plus one sample at start and stop), or
    `nvidia-smi -lms 100` when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    NVML_REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.rows = []  # (sm_mhz, max_mhz, power_w, reasons set)
        self.proc = None
        self.thread = None
        self.stop_evt = threading.Event()
        self.nvml = None
        self.handle = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(device).uuid)
                self.handle = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(device)
        except Exception:
            self.nvml = None

    def _sample_nvml(self):
        n, h = self.nvml, self.handle
        try:
            sm = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
            mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
            pw = n.nvmlDeviceGetPowerUsage(h) / 1000.0
            bits = n.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.rows.append((float(sm), float(mx), pw, {k for k, b in self.NVML_REASONS.items() if bits & b}))
        except Exception:
            pass

    def start(self):
        if self.nvml is not None:
            self._sample_nvml()

            def loop():
                while not self.stop_evt.wait(0.01):
                    self._sample_nvml()

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i",
                 str(self.device), "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                self.rows.append((float(parts[0]), float(parts[1]), float(parts[2]),
                                  {nm for nm, v in zip(names, parts[4:8]) if v.lower().startswith("active")}))
            except ValueError:
                pass

    def stop(self):
        self.stop_evt.set()
        if self.nvml is not None:
            if self.thread:
                self.thread.join(timeout=2)
            self._sample_nvml()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)
        return self.summary()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        reasons = set()
        for r in self.rows:
            reasons |= r[3]
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(reasons), "samples": len(self.rows),
                "power_w_max": max(r[2] for r in self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference_run(x, w, workers: int):
    """One run of the reference engine (oracle/_ref) or, if it was not built,
    the C restatement (oracle), on the host cores. Returns (seconds, kind)."""
    import oracle
    cfg = w.config.to_c()
    cfg.workers = workers
    if oracle.ref_available():
        r = oracle.ref_run(x, cfg, w.normalized)
        return r["run_ms"] / 1e3, "reference", r
    t0 = time.perf_counter()
    r = oracle.oracle_run(x, cfg, w.normalized)
    return time.perf_counter() - t0, "port", r


KERNEL_TIMING = ("CUDA events around each launch on the engine's stream, in an instrumented pass of the same K steps "
                 "run right after the timed ones (engine option kernel_events; off in the timed steps)")


def bench_config(w):
    """The `config` object of the JSON line: identical in both arms."""
    return {"workload": w.name, "n": w.n, "d": w.d, "description": w.description,
            "l2": "a 512 MiB buffer written, then read back, between timed steps (cold, clean L2)"}


def cpu_sample_rows(w):
    """Rows the CPU reference runs on: the full input, except config 4 whose
    full run takes ~25 min on 8 cores (its NoSeq merge is 1.8e11 tests):
    there the first 400k rows (~30 s of CPU work) stand in as the sample."""
    return min(w.n, 400_000) if w.kind == 4 and w.n > 400_000 else w.n


def run_reference_arm(args):
    """The reference's own CPU path (oracle/_ref: the unmodified reference
    engine compiled from /root/reference) on this box's host cores. Loads no
    product library: the input comes from the same header-only generator
    compiled into oracle/_ref (include/skyline_baseline_gen.h)."""
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    import oracle
    from paper_2411_14968_b200.configs import make_config  # pure Python (no library load)
    w = make_config(args.config, args.n)
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libskyref.so was not built"}), flush=True)
        return 0
    x = oracle.ref_generate_baseline(w.kind, w.n, w.d, 42)
    ns = cpu_sample_rows(w)
    if ns < w.n:
        x = x[:ns].copy()
    cores = oracle.ref_lib().skyref_hardware_concurrency()
    # each step is one full-size skyline::run; the number of runs is capped
    # so the arm ends within a few minutes on slow configs (config 4: ~25 min
    # per run on 8 cores -> 1 run)
    budget_s = float(os.environ.get("SKY_REF_BUDGET_S", "150"))
    times = []
    kind = None
    t_start = time.perf_counter()
    warm = args.warmup
    i = 0
    while len(times) < args.steps:
        t, kind, r = cpu_reference_run(x, w, cores)
        if i >= warm or (i == 0 and t * (args.warmup + args.steps) > budget_s):
            # slow run: it counts as the first timed step (no further warm-up)
            warm = min(warm, i)
            times.append(t)
        i += 1
        if time.perf_counter() - t_start + t > budget_s and times:
            break
    total = sum(times)
    value = ns * len(times) / total
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "warmup": warm, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generators, seed 42)",
        "config": bench_config(w),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": (f"full workload (N={w.n})" if ns == w.n else f"first {ns} of {w.n} rows")
                                   + f", {len(times)} timed runs of skyline::run "
                                   f"(requested {args.steps}; capped at ~{budget_s:.0f} s), workers={cores}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "skyline_size": int(r["final_size"]), "requested_steps": args.steps,
        "phase_ms": {"partition": r["partition_ms"], "local": r["local_ms"], "merge": r["merge_ms"]},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2411_14968_b200 import Engine
    from paper_2411_14968_b200.configs import make_config
    from paper_2411_14968_b200.skyline import generate

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    w = make_config(args.config, args.n)
    x = generate(w.kind, w.n, w.d, 42)
    # multi-GPU: rank r holds rows [N*r/W, N*(r+1)/W) (its shard, in HBM for
    # `value`, in pinned host memory for `e2e`) and calls sky_run_shard
    r0, r1 = w.n * rank // world, w.n * (rank + 1) // world
    x_mine = x[r0:r1] if world > 1 else x
    x_pin = torch.from_numpy(np.ascontiguousarray(x_mine)).pin_memory()
    x_host = x_pin.numpy()  # pinned view
    x_dev = x_pin.to(f"cuda:{local}")
    if world > 1:
        # one query sharded over the ranks: NCCL communicator inside the engine
        from paper_2411_14968_b200 import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng = Engine.distributed(local, rank, world, obj[0])
    else:
        eng = Engine(local)
    stream = torch.cuda.current_stream()
    eng.set_stream(stream.cuda_stream)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    flush_i32 = flush.view(torch.int32)
    n, d = x.shape
    n_mine = x_mine.shape[0]

    def step_dev():
        if world > 1:
            return eng.run_shard(None, w.config, w.normalized, device_ptr=x_dev.data_ptr(), n=n_mine, d=d)
        return eng.run(None, w.config, w.normalized, device_ptr=x_dev.data_ptr(), n=n, d=d)

    def step_e2e():
        if world > 1:
            return eng.run_shard(x_host, w.config, w.normalized)
        return eng.run(x_host, w.config, w.normalized)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        r = step_dev()
    if not args.no_e2e:
        step_e2e()

    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def timed(fn):
        ms = []
        res = []
        for k in range(args.steps):
            flush.fill_(k & 0xFF)  # > L2: evicts the previous step's lines
            # read it back: the fill leaves L2 full of dirty lines whose
            # write-back would otherwise land inside the next timed step
            flush_i32.max()
            torch.cuda.synchronize()
            barrier()
            ev0.record(stream)
            res.append(fn())
            ev1.record(stream)
            ev1.synchronize()
            ms.append(ev0.elapsed_time(ev1))
            if len(res) > 1:
                # every step must return the same ids; the previous step's id
                # array is then dropped (a caller does not hoard results, and
                # the library reuses the buffer), its metrics are kept
                assert np.array_equal(res[-2].skyline, res[-1].skyline), "non-deterministic skyline across steps"
                res[-2].skyline = None
            barrier()
        torch.cuda.synchronize()
        return ms, res

    clocks = ClockSampler(local)
    clocks.start()
    dev_ms, dev_res = timed(step_dev)
    e2e_ms, e2e_res = (None, None) if args.no_e2e else timed(step_e2e)
    # Per-kernel durations (the roofline's denominators) come from a second,
    # instrumented pass of the same steps: CUDA events recorded around every
    # dominance launch and HBM pass. The records sit between kernels and cost
    # 25-55 us per step, so the timed passes above run without them.
    eng.set_option("kernel_events", 1)
    step_dev()
    _, prof_res = timed(step_dev)
    eng.set_option("kernel_events", 0)
    clk = clocks.stop()

    total_dev = sum(dev_ms)
    total_e2e = sum(e2e_ms) if e2e_ms else None
    if world > 1:
        t = torch.tensor([total_dev, total_e2e or 0.0], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_dev, total_e2e = float(t[0]), (float(t[1]) if total_e2e is not None else None)

    # one query per step over all ranks (strong scaling): each rank's local
    # and merge phases cover its shard; every rank returns the full result
    jobs = 1
    r = dev_res[-1]
    m = r.metrics
    value = w.n * args.steps * jobs / (total_dev / 1e3)
    tests_per_step = statistics.mean(rr.metrics.tests_total for rr in dev_res)
    dom_ms = statistics.mean(rr.metrics.dom_kernel_ms for rr in prof_res)
    dom_tests = statistics.mean(rr.metrics.dom_tests for rr in dev_res)
    launches = sum(rr.metrics.kernel_launches for rr in dev_res)
    if world > 1:
        t = torch.tensor([launches], dtype=torch.int64, device=f"cuda:{local}")
        dist.all_reduce(t)
        launches = int(t[0])

    peaks = measured_peaks()
    props = torch.cuda.get_device_properties(local)
    n_sm = props.multi_processor_count
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    # 1 dominance test = d FP32 compares, peak 64 compares/clk/SM.
    # The packed-code test evaluates d attributes in ~3.5 instructions, so that
    # ratio may exceed 1 (SURVEY 8(d) anticipates it); the roofline is the
    # packed test's own measured issue peak, the compare ratio rides along.
    tests_s = dom_tests / (dom_ms / 1e3) if dom_ms > 0 else 0.0
    achieved = tests_s * d / 1e9  # Gcompare/s
    peak = n_sm * FP32_COMPARES_PER_CLK_PER_SM * sm_max * 1e6 / 1e9
    per_clk = PACKED_TESTS_PER_CLK_PER_SM if d <= 16 else FP32_COMPARES_PER_CLK_PER_SM / d
    ipeak_model = n_sm * per_clk * sm_max * 1e6
    # measured: the dominance core's packed-code test loop alone on every SM
    # (sky_issue_peak, k_issue_peak), outside the timed region
    ipeak_meas = eng.issue_peak(d) if d <= 16 else None
    ipeak = ipeak_meas or ipeak_model
    traffic, traffic_src = ncu_traffic(f"c{args.config}")
    # the roofline of the dominance kernels is the packed test's own issue
    # peak (measured); SURVEY 8(d)'s FP32-compare figure rides along, and its
    # ratio exceeds 1 because one packed test stands for d compares
    roofline = {
        "bound": "alu", "kernel": "k_relsky3 + k_bnl2 (dominance tests)", "achieved": tests_s / 1e9,
        "peak": ipeak / 1e9, "unit": "Gtest/s", "frac": tests_s / ipeak if ipeak else None, "traffic": traffic,
        "traffic_source": traffic_src,
        "algorithmic_unit": f"1 dominance (pair) test of d = {d} attributes",
        "peak_source": ("measured: k_issue_peak (the packed-code test loop of k_relsky3 alone, every SM, "
                        "best of K in {4,8} x 2..8 CTAs/SM; sky_issue_peak); operands in shared memory, "
                        "no HBM/tensor term" if ipeak_meas else "model"),
        "model_peak_gtest_s": ipeak_model / 1e9,
        "model": ("d<=16: 2 IMAD (fma pipe) + 1 LOP3 + 1/2 VIMNMX3 (alu pipe) per test, fma/alu pipes 2 cyc "
                  "per warp instruction -> 32 tests/clk/SM" if d <= 16 else
                  f"d>16: {d} FP32 compares per test -> 64/{d} tests/clk/SM"),
        "scalar_compares": {
            "achieved_gcompare_s": achieved, "peak_gcompare_s": peak,
            "ratio": achieved / peak if peak else None,
            "unit": f"1 test = d = {d} FP32 compares (SURVEY 8(d))",
            "peak_source": f"{n_sm} SM x {FP32_COMPARES_PER_CLK_PER_SM} FP32 compare/clk x sm_max_mhz {sm_max} "
                           "(MEASURED_PEAKS.json clock)",
        },
        "kernel_ms_per_step": dom_ms, "kernel_share_of_step": dom_ms / statistics.mean(dev_ms),
        "kernel_timing": KERNEL_TIMING,
        "tests_per_step": dom_tests,
        "ncu_pipe_mix": ncu_pipe_mix(f"c{args.config}"),
    }

    # HBM streaming passes (prep, representative prefilter, candidate pass):
    # algorithmic bytes (rows read once, keys written/read) / CUDA-event time
    s_ms = statistics.mean(rr.metrics.stream_kernel_ms for rr in prof_res)
    s_bytes = statistics.mean(rr.metrics.stream_bytes for rr in dev_res)
    hbm_peak = peaks.get("hbm_gbs", 6553.6)
    s_gbs = s_bytes / (s_ms / 1e3) / 1e9 if s_ms > 0 else 0.0
    s_traffic, s_traffic_src = ncu_stream_traffic(f"c{args.config}")
    hbm_passes = {
        "bound": "hbm", "kernel": "k_prep_stream / k_prep + k_prefilter (+ k_cand_bucket on the stream path)",
        "achieved": s_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": s_gbs / hbm_peak if hbm_peak else None,
        "traffic": s_traffic, "traffic_source": s_traffic_src,
        "algorithmic_bytes_per_step": s_bytes, "kernel_ms_per_step": s_ms,
        "kernel_share_of_step": s_ms / statistics.mean(dev_ms),
        "kernel_timing": KERNEL_TIMING,
        "launches_per_step": statistics.mean(rr.metrics.stream_launches for rr in dev_res),
        "algorithmic_unit": "per row: prep 4d B read + 8-12 B written; prefilter 4d B read (stream path; the staged keys, read only with codes, not counted) or "
                            "4d + 5 B (sorted path); candidate pass 8 B read",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if "hbm_gbs" in peaks else
                       "B200_PROFILING.md fallback",
    }
    if s_ms > dom_ms:
        # the streaming passes dominate the step (e.g. config 3): they are the roofline
        hbm_passes["dominance_kernels"] = roofline
        roofline = hbm_passes
    else:
        roofline["hbm_passes"] = hbm_passes

    line = {
        "metric": BASELINE_METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": total_dev / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (sky_generate, seed 42)",
        "config": bench_config(w),
        "effective_p": r.effective_p,
        "parallelism": (f"{world} ranks: rows sharded (partition + representative prefilter per shard), "
                        "survivors routed to partition owners (NCCL all-to-all), local skylines all-gathered, "
                        "candidate-sharded merge") if world > 1 else "single-gpu",
        "tests_per_s": tests_per_step * args.steps * jobs / (total_dev / 1e3),
        "skyline_size": int(r.skyline.size), "union_size": m.union_size, "filtered_count": m.filtered_count,
        "phase_ms": {"partition": m.partition_ms, "local": m.local_ms, "merge": m.merge_ms},
        "tests_per_step": {"reps_prefilter": m.tests_reps, "local": m.tests_local, "merge": m.tests_merge,
                           "exact_checks": m.dom_exact_checks},
        "roofline": roofline,
        "clocks": clk,
        "gpu_launches": launches,
    }
    if total_e2e is not None:
        e0 = e2e_res[-1]
        assert np.array_equal(e0.skyline, r.skyline)
        h2d, d2h = int(e0.metrics.h2d_bytes), int(e0.metrics.d2h_bytes)
        if world > 1:  # every rank copies its own shard in and the ids out
            t = torch.tensor([h2d, d2h], dtype=torch.int64, device=f"cuda:{local}")
            dist.all_reduce(t)
            h2d, d2h = int(t[0]), int(t[1])
        line["e2e"] = {"value": w.n * args.steps * jobs / (total_e2e / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "ms_per_step": total_e2e / args.steps}
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        ns = cpu_sample_rows(w)
        xs = x if ns == w.n else np.ascontiguousarray(x[:ns])
        t, kind, rr = cpu_reference_run(xs, w, os.cpu_count() or 1)
        cores = os.cpu_count() or 1
        if kind == "reference":
            cores = oracle.ref_lib().skyref_hardware_concurrency()
        if ns == w.n:
            assert np.array_equal(rr["ids"], r.skyline), "GPU skyline differs from the CPU reference"
            parity = "ids identical"
        else:
            parity = "sample run (full-size parity: tests/test_full_size.py goldens)"
        line["cpu_baseline"] = {"value": ns / t, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": (f"full workload (N={w.n})" if ns == w.n else
                                           f"first {ns} of the {w.n} rows (a full run takes ~25 min on 8 cores)")
                                + f", 1 run of skyline::run, workers={cores}",
                                "ms": t * 1e3, "parity": parity}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
