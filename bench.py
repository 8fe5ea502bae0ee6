#!/usr/bin/env python
"""Benchmark: 4-bit GREEDY row-wise quantization (b=200, r=0.16) of a 20M x 64 fp32 table.

BASELINE.json metric: "rows/sec and GB/s for 4-bit GREEDY rowwise quant
(20M x 64 fp32); % roofline" on config 5b (20,000,000 x 64, mixed
"trained-embedding" distribution).  One step = one fused pass of the hot path
(clip search + quantize + nibble pack + fp16 scale/bias) over the whole table
resident in HBM.  Prints ONE JSON line (rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one process per GPU; every rank quantizes its own
20M-row table (rows are independent: weak scaling, no collective on the data
path) and the step time is the max over ranks.  ``--impl reference`` times the
reference algorithm on the host CPU (the C restatement in oracle/, all host
threads) on a bounded sample of the same workload.
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

METRIC = "rows/sec and GB/s for 4-bit GREEDY rowwise quant (20M×64 fp32); % roofline"
ROWS, DIM, B, R, AUX = 20_000_000, 64, 200, 0.16, "fp16"
FLOP_PER_ELEM_EVAL = 13   # table.py:100-103 literal ops


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes ~0.1-0.5 s to emit its first sample: start the timed region only
            # once it is sampling, so the samples cover the whole region
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.005)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_reference_rate(rows_sample: int, seed: int = 1911, steps: int = 1, warmup: int = 0):
    """GREEDY b=200 r=0.16 fp16 on the host (oracle C port, all threads): rows/s."""
    import oracle
    from oracle import rng

    x = rng.mixed_table(rows_sample, DIM, seed)
    nthreads = oracle.max_threads()
    for _ in range(warmup):
        oracle.quantize_pack_table(x[: max(1, rows_sample // 10)], "greedy", B, R, AUX, nthreads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.quantize_pack_table(x, "greedy", B, R, AUX, nthreads)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    return rows_sample / t, nthreads, t


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _ref_chunk(args):
    """One chunk through the unmodified reference package (baseline/_ref): packed bytes."""
    path, x, method = args
    if path not in sys.path:
        sys.path.insert(0, path)
    import embquant

    t = embquant.EmbeddingTable(x)
    q = embquant.quantize_table(t, method, 4, AUX, b=B, r=R)
    return embquant.pack_table4(q).buffer.tobytes()


def python_reference_rate(rows: int = 10_000, seed: int = 1911):
    """Context only: the UNMODIFIED Python reference -- the reference
    package pip-installed into baseline/_ref from the reference tree -- timed on the bench's
    mixed generator, GREEDY b=200 r=0.16 fp16, one process per host core over row chunks.
    Its bytes are checked against the oracle.  None when baseline/_ref is absent."""
    import multiprocessing as mp

    import oracle
    from oracle import rng

    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "embquant")):
        return None
    x = rng.mixed_table(rows, DIM, seed)
    procs = os.cpu_count() or 1
    chunks = [(path, x[i::procs].copy(), "greedy") for i in range(procs)]
    with mp.get_context("spawn").Pool(procs) as pool:
        pool.map(_ref_chunk, [(path, x[:procs], "greedy")] * procs)   # warm the workers
        t0 = time.perf_counter()
        parts = pool.map(_ref_chunk, chunks)
        t = time.perf_counter() - t0
    want = oracle.quantize_pack_table(x, "greedy", B, R, AUX)
    stride = (DIM + 1) // 2 + 4
    got = np.empty((rows, stride), np.uint8)
    for i, part in enumerate(parts):
        got[i::procs] = np.frombuffer(part, np.uint8).reshape(-1, stride)
    return {"value": rows / t, "unit": "rows/s", "cores": procs, "kind": "reference",
            "sample": f"{rows} rows x {DIM} mixed, GREEDY b=200 r=0.16 fp16, unmodified reference "
                      f"package (baseline/_ref) in {procs} processes, {t:.2f} s",
            "bytes_match_oracle": bool(np.array_equal(got.reshape(-1), want.packed))}


def parity_report(eq, torch, dev, x, out, method, b, sample=0, x_host=None, nthreads=0):
    """Check a timed launch's packed bytes against the CPU oracle on the same table.

    x (device, rows x d) is the timed input and ``out`` the timed launch's packed output
    (left untouched); per-row float64 ranges come from one more, untimed launch into a
    scratch buffer.  ``sample`` = 0 checks every row, else a strided sample of that many
    rows (first and last included).  GREEDY adds the reference's own near-ties from the
    oracle's walk (relative gap < 1e-6 between the two competing losses, clipping.py:185,
    and between candidate and best, :187,191) and the kernel's float64 re-decision count;
    HIST-BRUTE counts windows that differ only at a norm tie (<= 1e-12 relative).  Run
    outside every timed region; the oracle is the checker, not the thing measured."""
    import oracle
    import numpy as np

    rows, d = int(x.shape[0]), int(x.shape[1])
    stride = eq.packed_row_stride(d, AUX)
    t0 = time.perf_counter()
    rr = eq.RowResults(torch.empty(rows, dtype=torch.float64, device=dev),
                       torch.empty(rows, dtype=torch.float64, device=dev),
                       torch.empty(rows, dtype=torch.int32, device=dev),
                       torch.empty(rows, dtype=torch.int32, device=dev),
                       torch.empty(rows, dtype=torch.float64, device=dev))
    from paper_1911_02079_b200 import _lib

    _lib.diag_counters(reset=True)
    scratch = torch.empty(rows * stride, dtype=torch.uint8, device=dev)
    eq.quantize_pack_table4(x, method, AUX, b, R, out=scratch, rows_out=rr)
    diag = _lib.diag_counters(reset=True)
    same_as_timed = bool(torch.equal(scratch, out.view(-1)[: rows * stride]))
    del scratch
    if sample and sample < rows:
        idx = torch.unique(torch.cat([torch.arange(0, rows, max(1, rows // sample), device=dev),
                                      torch.tensor([rows - 1], device=dev)]))
    else:
        idx = None
    sel = (lambda t: t) if idx is None else (lambda t: t[idx])
    got = sel(out.view(rows, stride)).cpu().numpy()
    glo, ghi = sel(rr.xmin).cpu().numpy(), sel(rr.xmax).cpu().numpy()
    gi0, gi1 = sel(rr.info0).cpu().numpy(), sel(rr.info1).cpu().numpy()
    if x_host is not None and idx is None:
        xs = x_host
    else:
        xs = sel(x).cpu().numpy()
    nthreads = nthreads or oracle.max_threads()
    rep = {"rows_checked": int(xs.shape[0]), "of_rows": rows, "method": method}
    if method == "greedy":
        want, g_lr, g_best = oracle.quantize_pack_table_gaps(xs, b, R, AUX, nthreads)
    else:
        want = oracle.quantize_pack_table(xs, method, b, R, AUX, nthreads)
    bad_bytes = np.nonzero((got != want.packed.reshape(-1, stride)).any(axis=1))[0]
    bits = lambda a: np.ascontiguousarray(a, np.float64).view(np.uint64)
    bad_range = np.nonzero((bits(glo) != bits(want.xmin)) | (bits(ghi) != bits(want.xmax)))[0]
    rep["byte_mismatches"] = int(bad_bytes.size)
    rep["range_mismatches"] = int(bad_range.size)
    if method == "greedy":
        rep["near_ties_lr"] = int(np.sum(g_lr < 1e-6))
        rep["near_ties_best"] = int(np.sum(g_best < 1e-6))
        bad = np.union1d(bad_bytes, bad_range)
        # the only exception north_star permits: the reference's two competing losses within 1e-6
        rep["excused_lr_ties"] = int(np.sum(g_lr[bad] < 1e-6)) if bad.size else 0
        it = np.where(gi0 >= 0, gi0, 0).astype(np.int64)
        rep["iterations_match"] = bool(np.array_equal(np.where(want.info0 >= 0, want.info0, 0), it))
        rep["exact_redecisions"] = diag["exact_redecisions"]
        rep["exact_code_rows"] = diag["exact_code_rows"]
        rep["redecisions_over_rows"] = rows
    if method == "hist-brute":
        ties = 0
        for i in np.union1d(bad_bytes, bad_range):
            ng = oracle.hist_window_norm(xs[i], b, int(gi0[i]), int(gi1[i]))
            no = oracle.hist_window_norm(xs[i], b, int(want.info0[i]), int(want.info1[i]))
            if abs(ng - no) <= 1e-12 * max(abs(ng), abs(no)):
                ties += 1
        rep["hist_ties"] = ties
    rep["launch_bytes_reproduced"] = same_as_timed
    rep["oracle_threads"] = nthreads
    rep["check_s"] = round(time.perf_counter() - t0, 2)
    return rep


def run_reference(args, rank: int):
    if rank != 0:
        return
    sample = args.cpu_rows
    rate, cores, t = cpu_reference_rate(sample, steps=args.steps, warmup=min(args.warmup, 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "rows/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "GREEDY b=200 r=0.16 fp16-aux, 20M x 64 mixed (config 5b); "
                               f"each step a {sample}-row sample on the host",
                   "rows": ROWS, "dim": DIM, "b": B, "r": R, "aux": AUX},
        "cpu_baseline": {"value": rate, "unit": "rows/s", "cores": cores, "kind": "port",
                         "cpu_model": _cpu_model(),
                         "sample": f"{sample} rows x {DIM} of the mixed generator "
                                   "(oracle/eq4_oracle.c restatement of the reference, "
                                   f"{cores} OpenMP threads)"},
        "e2e": {"value": rate, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank: int, world: int):
    import torch

    import paper_1911_02079_b200 as eq
    from paper_1911_02079_b200 import workloads

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rows = args.rows
    stride = eq.packed_row_stride(DIM, AUX)
    x = workloads.mixed_table(rows, DIM, seed=1911 + rank, device=dev)
    out = torch.empty(rows * stride, dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        eq.quantize_pack_table4(x, "greedy", AUX, B, R, out=out, status=status, stream=stream,
                                check=False)

    # algorithmic work: per-row loss evaluations from one untimed launch
    rr = eq.RowResults(None, None, torch.empty(rows, dtype=torch.int32, device=dev), None, None)
    eq.quantize_pack_table4(x, "greedy", AUX, B, R, out=out, rows_out=rr, stream=stream)
    it = rr.info0.to(torch.int64)
    evals = int(torch.where(it >= 0, 1 + 2 * it, torch.zeros_like(it)).sum().item())
    del rr, it
    flop_per_step = float(FLOP_PER_ELEM_EVAL) * DIM * evals
    bytes_per_step = float(rows) * (4 * DIM + (DIM + 1) // 2 + 4)

    for _ in range(args.warmup):
        step()
    dist = world > 1
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    st = int(status.item())
    if st:
        raise SystemExit(f"kernel status {st}: data error in the bench table")
    if dist:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = world * rows / (ms * 1e-3)

    # end to end through the public API: pinned host table in, packed bytes out
    e2e = None
    parity = None
    if not args.no_parity:
        # the timed bytes against the oracle on the same table (every row at N = 1)
        psample = args.parity_rows if args.parity_rows >= 0 else (0 if world == 1 else 1_000_000)
        parity = parity_report(eq, torch, dev, x, out, "greedy", B, sample=psample)
    if not args.no_e2e:
        # every rank pins its own table + output; all ranks agree before any collective
        ok, why = 1, ""
        try:
            xh = torch.empty((rows, DIM), dtype=torch.float32, pin_memory=True)
            oh = torch.empty(rows * stride, dtype=torch.uint8, pin_memory=True)
        except RuntimeError as ex:
            ok, why = 0, f"pinned host allocation failed: {ex}".splitlines()[0]
        if dist:
            okt = torch.tensor([ok], device=dev)
            torch.distributed.all_reduce(okt, op=torch.distributed.ReduceOp.MIN)
            ok = int(okt.item())
        if not ok:
            e2e = {"value": None, "unit": "rows/s", "h2d_bytes_per_step": rows * DIM * 4,
                   "d2h_bytes_per_step": rows * stride, "error": why or "a rank could not pin its table"}
    if not args.no_e2e and e2e is None:
        xh.copy_(x)
        table = eq.EmbeddingTable(xh.numpy())   # validated once, like the reference's constructor
        # context for the e2e number: one plain pinned H2D copy of the whole table (the PCIe floor)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        x.copy_(xh, non_blocking=True)
        torch.cuda.synchronize(dev)
        h2d_gbps = rows * DIM * 4 / (time.perf_counter() - t0) / 1e9
        del x
        torch.cuda.empty_cache()
        outh = oh.numpy()
        eq.quantize_pack_table4(table, "greedy", AUX, B, R, out=outh)
        if dist:
            torch.distributed.barrier()
        e_steps = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            eq.quantize_pack_table4(table, "greedy", AUX, B, R, out=outh)
        te = (time.perf_counter() - t0) / e_steps
        if dist:
            tt = torch.tensor([te], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": world * rows / te, "unit": "rows/s", "ms_per_step": te * 1e3,
               "h2d_bytes_per_step": rows * DIM * 4, "d2h_bytes_per_step": rows * stride,
               "path": "quantize_pack_table4(EmbeddingTable(pinned host), 'greedy', 'fp16') -> "
                       "eq4_quantize_pack_host (chunked H2D/kernel/D2H overlap)",
               "h2d_GBps_plain_copy": h2d_gbps,
               "h2d_floor_ms": rows * DIM * 4 / (h2d_gbps * 1e9) * 1e3}

    if rank != 0:
        return
    peaks = _peaks()
    props = torch.cuda.get_device_properties(dev)
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = props.multi_processor_count * 128 * 2 * sm_max * 1e6 / 1e12
    peak_source = ("derived: SMs x 128 FP32 lanes x 2 x sm_max_mhz (no measured FP32 figure found)")
    mp = os.path.join(ROOT, "profiles", "r02_fp32_peak.json")
    if os.path.exists(mp):
        with open(mp) as f:
            fp32_peak = float(json.load(f)["peak_used"])
        peak_source = ("measured: profiles/r02_fp32_peak.json, FFMA2 throughput of this B200 model "
                       "(tools/microbench/fp32_peak.cu; MEASURED_PEAKS.json has no FP32 figure)")
    achieved = flop_per_step / (ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("greedy_20Mx64", {}).get("dram_bytes_per_launch")
    cpu = None
    if not args.no_cpu and world == 1:   # the reported CPU baseline: rank 0 at N = 1 only
        rate, cores, t = cpu_reference_rate(args.cpu_rows)
        cpu = {"value": rate, "unit": "rows/s", "cores": cores, "kind": "port",
               "cpu_model": _cpu_model(),
               "sample": f"{args.cpu_rows} rows x {DIM} mixed, GREEDY b=200 r=0.16 fp16 "
                         f"(oracle C restatement, {cores} threads, {t:.1f} s)"}
        try:
            cpu["python_reference_context"] = python_reference_rate()
        except Exception as ex:   # context only: never fails the bench
            cpu["python_reference_context"] = {"error": str(ex).splitlines()[0][:200]}
    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (f64 exact re-decisions)", "data": "synthetic",
        "config": {"workload": "GREEDY b=200 r=0.16 fp16-aux on 20,000,000 x 64 fp32 (config 5b, "
                               "mixed trained-embedding generator) per GPU",
                   "rows_per_gpu": rows, "dim": DIM, "b": B, "r": R, "aux": AUX,
                   "l2": "input 5.12 GB per GPU >> 126 MB L2 (no flush needed)",
                   "parallelism": f"row-sharded x{world}, no data-path collective"},
        "input_GBps": world * rows * DIM * 4 / (ms * 1e-3) / 1e9,
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp32_peak, "traffic": traffic,
                     "peak_source": peak_source,
                     "work": f"13 FLOP x d x loss evaluations ({evals} evals/step)",
                     "hbm_floor_ms": bytes_per_step / (float(peaks.get('hbm_gbs', 6546.9)) * 1e9) * 1e3,
                     "pipes_ncu": ncu_pipes()},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "parity": parity,
        "gpu_launches": args.steps,
        "clocks": clocks.summary(),
    }
    if args.secondary and world == 1:   # the other configs are single-GPU lines
        line["secondary"] = secondary(eq, workloads, torch, dev, peaks, fp32_peak, check=not args.no_parity)
        line["secondary"]["sls_20Mx64_greedy_packed"] = sls_secondary(eq, torch, dev, peaks, out, rows)
    print(json.dumps(line), flush=True)


def ncu_pipes():
    """FMA-pipe, ALU-pipe and issue utilisation of the screening kernel on this workload, from the
    committed ncu capture (a separate profiled launch, not the timed run -- context for `roofline`).
    An FFMA2 / FADD2 holds its issue slot for two cycles (K2), so `issue_slots_pct` adds
    the packed instructions' second cycle to ncu's issued-instruction count."""
    path = os.path.join(ROOT, "profiles", "r02_greedy_fast_20Mx64_issue_slots.json")
    try:
        with open(path) as fh:
            j = json.load(fh)
    except (OSError, ValueError):
        return None
    out = {k: j.get(k) for k in ("kernel", "fma_pipe_pct", "alu_pipe_pct", "issue_active_pct", "issue_slots_pct")}
    out["source"] = "profiles/r02_greedy_fast_20Mx64_issue_slots.json (ncu --set full, one launch, not the timed run)"
    return out


def _time_method(eq, torch, dev, x, method, b, n=10, warm=3, parity=None, parity_sample=0):
    """Device time (CUDA events on the current stream) of one fused launch over x, plus the
    GREEDY loss-evaluation count of that launch (clipping.py:174,183-184) for the roofline."""
    rows, d = x.shape
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.empty(rows * eq.packed_row_stride(d, AUX), dtype=torch.uint8, device=dev)
    evals = None
    if method == "greedy":
        rr = eq.RowResults(None, None, torch.empty(rows, dtype=torch.int32, device=dev), None, None)
        eq.quantize_pack_table4(x, method, AUX, b, R, out=out, rows_out=rr)
        it = rr.info0.to(torch.int64)
        evals = int(torch.where(it >= 0, 1 + 2 * it, torch.zeros_like(it)).sum().item())
        del rr, it
    f = lambda: eq.quantize_pack_table4(x, method, AUX, b, R, out=out, status=st, check=False)
    for _ in range(warm):
        f()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize(dev)
    if int(st.item()):
        raise SystemExit(f"kernel status {int(st.item())} in a secondary workload ({method})")
    ms = e0.elapsed_time(e1) / n
    if parity is not None:   # the timed launches' bytes against the oracle (untimed)
        parity.update(parity_report(eq, torch, dev, x, out, method, b, sample=parity_sample))
    del out
    return ms, evals


def secondary(eq, workloads, torch, dev, peaks, fp32_peak, check=True):
    """The other BASELINE.json configs, device-timed (each table >> L2 or re-read per launch):
    config 2 (ASYM 4M x 64, HBM-bound), config 3 (GREEDY 4M x 128 mixed), config 4 (HIST-BRUTE
    16,384 x 64), config 5a (GREEDY d-sweep over 1 GiB N(0,1) tables), plus the HIST-APPRX, ACIQ
    and GSS searches and row-wise KMEANS (§8f.4) on representative tables."""
    hbm = float(peaks.get("hbm_gbs", 6546.9))
    res = {}

    def greedy_line(x, d, ms, evals):
        rows = x.shape[0]
        flop = float(FLOP_PER_ELEM_EVAL) * d * evals
        return {"ms": ms, "rows_per_s": rows / ms * 1e3,
                "GBps": rows * (4 * d + (d + 1) // 2 + 4) / ms / 1e6,
                "alg_TFLOPs": flop / ms / 1e9, "fp32_frac": flop / ms / 1e9 / fp32_peak}

    x = workloads.gaussian_table(4_194_304, 64, 7, device=dev)
    par = {} if check else None
    ms, _ = _time_method(eq, torch, dev, x, "asym", B, parity=par, parity_sample=0)
    byt = 4_194_304 * (4 * 64 + 32 + 4)
    res["asym_4Mx64_config2"] = {"ms": ms, "rows_per_s": 4_194_304 / ms * 1e3, "GBps": byt / ms / 1e6,
                                 "hbm_frac": byt / ms / 1e6 / hbm, "parity": par}
    del x
    x = workloads.mixed_table(4_194_304, 128, 7, device=dev)
    par = {} if check else None
    ms, ev = _time_method(eq, torch, dev, x, "greedy", B, parity=par, parity_sample=1_000_000)
    res["greedy_4Mx128_mixed_config3"] = dict(greedy_line(x, 128, ms, ev), parity=par)
    del x
    # config 4: HIST-BRUTE b=200 (compute-bound, no roofline target): per-row time and the
    # reference's bin-visit counter rate (histclip.py:162-164)
    x = workloads.gaussian_table(16384, 64, 7, device=dev)
    par = {} if check else None
    ms, _ = _time_method(eq, torch, dev, x, "hist-brute", 200, n=5, warm=2, parity=par, parity_sample=0)
    visits = 16384 * 200 * (200 * 201 // 2)
    # the reference's bin-visit counter: the pruned kernel scores only a few % of the windows
    res["hist_brute_16384x64_config4"] = {"ms": ms, "us_per_row": ms * 1e3 / 16384,
                                          "reference_equivalent_bin_visits_per_s": visits / ms * 1e3,
                                          "parity": par}
    # HIST-APPRX (histclip.py:181-217) on the same table: 2b - 1 = 399 window norms per row
    par = {} if check else None
    ms, _ = _time_method(eq, torch, dev, x, "hist-apprx", 200, n=5, warm=2, parity=par, parity_sample=0)
    res["hist_apprx_16384x64"] = {"ms": ms, "us_per_row": ms * 1e3 / 16384, "parity": par}
    del x
    # ACIQ (clipping.py:115-139): two numpy-order float64 sums per row + codes, bandwidth-class
    x = workloads.gaussian_table(4_194_304, 64, 7, device=dev)
    par = {} if check else None
    ms, _ = _time_method(eq, torch, dev, x, "aciq", B, parity=par, parity_sample=1_000_000)
    res["aciq_4Mx64"] = {"ms": ms, "GBps": byt / ms / 1e6, "hbm_frac": byt / ms / 1e6 / hbm,
                         "parity": par}
    del x
    # GSS (clipping.py:70-112): ~23 exact float64 quant_mse per row
    x = workloads.gaussian_table(1_048_576, 64, 7, device=dev)
    par = {} if check else None
    ms, _ = _time_method(eq, torch, dev, x, "gss", B, n=5, warm=2, parity=par, parity_sample=250_000)
    res["gss_1Mx64"] = {"ms": ms, "rows_per_s": 1_048_576 / ms * 1e3, "parity": par}
    del x
    # row-wise KMEANS codebooks (codebook.py:35-172), the EMBQ kmeans_row payload
    from paper_1911_02079_b200.codebook import kmeans_rows, kmeans_row_stride
    x = workloads.gaussian_table(262_144, 128, 7, device=dev)
    kout = torch.empty(262_144 * kmeans_row_stride(128, AUX), dtype=torch.uint8, device=dev)
    kit = torch.empty(262_144, dtype=torch.int32, device=dev)
    kmeans_rows(x, AUX, out=kout, iters=kit)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        kmeans_rows(x, AUX, out=kout, iters=kit, check=False)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / 5
    res["kmeans_rows_262144x128"] = {"ms": ms, "rows_per_s": 262_144 / ms * 1e3,
                                     "mean_lloyd_rounds": float(kit.clamp(min=0).float().mean().item())}
    del x, kout, kit
    # config 5a: GREEDY d-sweep, rows = 2^30 / (4 d): 1 GiB of fp32 per table
    sweep = {}
    for d in (16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192):
        rows = (1 << 30) // (4 * d)
        x = workloads.gaussian_table(rows, d, 7, device=dev)
        par = {} if check else None
        ms, ev = _time_method(eq, torch, dev, x, "greedy", B, n=5, warm=2, parity=par,
                              parity_sample=1_000_000)
        sweep[str(d)] = dict(greedy_line(x, d, ms, ev), parity=par)
        del x
    res["greedy_dsweep_1GiB_config5a"] = sweep
    return res


def sls_secondary(eq, torch, dev, peaks, packed_buf, rows, batch=16384, pool=64):
    """§8f.1 pooled lookup (sparse_lengths_sum_4bit) over the step's own GREEDY-packed
    20M x 64 fp16 table: batch x pool uniform random rows, timed as a CUDA graph of 20
    calls (no host gaps).  Algorithmic bytes = packed row + int64 index per pooled row
    + the fp32 output (bench.py:31-42 bytes model of the reference, plus index/output)."""
    p = eq.PackedTable4(rows, DIM, AUX, device_buffer=packed_buf)
    g = torch.Generator(device=dev).manual_seed(1911)
    idx = torch.randint(0, rows, (batch * pool,), device=dev, generator=g)
    ln = torch.full((batch,), pool, dtype=torch.int64, device=dev)
    q = eq.PooledQuery(idx, ln)
    o = torch.empty(batch, DIM, device=dev)
    eq.sparse_lengths_sum_4bit(p, q, out=o)   # validated once (raises on bad input)
    f = lambda: eq.sparse_lengths_sum_4bit(p, q, out=o, check=False)
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        for _ in range(3):
            f()
    torch.cuda.current_stream(dev).wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    n = 20
    with torch.cuda.graph(graph):
        for _ in range(n):
            f()
    graph.replay()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / n
    nrows = batch * pool
    alg = nrows * (eq.bytes_per_pooled_row("int4", DIM, AUX) + 8) + batch * DIM * 4
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get("sls_20Mx64", {}).get("dram_bytes_per_launch")
    return {"us": ms * 1e3, "batch": batch, "pooling": pool, "pooled_rows_per_s": nrows / ms * 1e3,
            "giga_sums_per_s": nrows * DIM / ms / 1e6, "alg_GBps": alg / ms / 1e6,
            "roofline": {"bound": "hbm", "achieved": alg / ms / 1e6,
                         "peak": float(peaks.get("hbm_gbs", 6546.9)), "unit": "GB/s",
                         "frac": alg / ms / 1e6 / float(peaks.get("hbm_gbs", 6546.9)),
                         "traffic": traffic,
                         "note": "random 36-byte row gathers: DRAM moves ~160 B per row"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--rows", type=int, default=ROWS)
    ap.add_argument("--cpu-rows", type=int, default=2_000_000)   # ~2 s x all host threads
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed bytes")
    ap.add_argument("--parity-rows", type=int, default=-1,
                    help="rows checked against the oracle (0 = all; default all at N = 1, 1M per rank above)")
    ap.add_argument("--secondary", action=argparse.BooleanOptionalAction, default=True,
                    help="config 2 ASYM, config 3 GREEDY and the SLS lookup, device-timed (rank 0)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        torch.distributed.init_process_group("nccl")
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
