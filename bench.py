"""Benchmark: detector shots/s of the sm_100a sampler vs the reference CPU sampler.

`python bench.py --gpus N --steps K --warmup W [--impl ours|reference] [--workload NAME]`

A step is one pass of the hot path over one batch of shots: Philox error
draw -> f = T.e -> direct parities -> autoregressive chain -> packed record
(for the 1e9-shot sweep workload: per-output counts). Each rank samples its
own disjoint global shot range (weak scaling; no data-path collective); with
N > 1 the per-output flip counts are all-reduced over NCCL once per step.

Timing: W untimed warm-up steps; K steps timed with CUDA events on the
launching stream, L2 flushed (256 MiB write) between steps outside the events;
barrier + synchronize around the timed region; max over ranks. `e2e` runs the
same shots through the C-ABI host entry (zxs_sample -> host record, D2H copy
inside the timed region). Rank 0 prints one JSON line.
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

WORKLOADS = {
    # name: (fixture path, BASELINE config index, description, default shots per GPU per step, count_only)
    "c2_surface_d3_xmem_t": ("tests/golden/c2_surface_d3_xmem_t.zxs", 1,
                             "d=3 rotated surface code X-memory, 3 rounds, p=1e-3, one T gate (chi=2)", 1 << 26, False),
    "c1_surface_d3_zmem": ("tests/golden/c1_surface_d3_zmem.zxs", 0,
                           "d=3 rotated surface code Z-memory, 3 rounds, p=1e-3, Clifford", 1 << 26, False),
    "c4_color_d5_rz3": ("tests/golden/c4_color_d5_rz3.zxs", 3,
                        "[[19,1,5]] colour code X-memory, 3 rounds, p=1e-3, R_Z on 3 data (chi=64)", 1 << 22, False),
    "c5_surface_d7_r7": ("tests/golden/c5_surface_d7_r7.zxs", 4,
                         "d=7 rotated surface code Z-memory, 7 rounds, p=1e-3, count-only sweep", 1 << 24, True),
    "c3_cultivation_proxy": ("data/c3_cultivation_proxy.zxs.gz", 2,
                             "Steane-code cultivation proxy: T injection + 2 transversal T checks (chi=46656)",
                             148 * 24576, False),  # one mono_kernel CTA tile (12 warps x 2048 shots) per SM
}
DEFAULT_WORKLOAD = "c2_surface_d3_xmem_t"


def _measured_hbm_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fp:
            return float(json.load(fp)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


MEASURED_HBM_GBS = _measured_hbm_gbs()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"\
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"\
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 5 + i and s[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------- reference arm
def reference_rate(path: str, target_s: float, seed: int, threads: int):
    """The reference's own sampler (oracle/_ref: proj/src compiled in place) on
    the host cores; falls back to the C restatement if the library is absent.
    Returns (shots/s, shots per call, kind, seconds)."""
    from oracle import coracle, refdriver
    if refdriver.available():
        m = refdriver.RefModel.load(path)

        def run(n):
            # SamplerOptions.batch_size (sampler.cpp:149-158): the reference default of 65536 shots,
            # lowered (in multiples of 64) only when a sample has fewer than threads x 65536 shots,
            # so every host thread gets a batch (workers = min(threads, batches)).
            bs = int(min(65536, max(64, (n // threads) // 64 * 64)))
            try:
                return m.sample(n, seed, batch_size=bs, threads=threads, force_dense=True)  # sample_detectors
            except RuntimeError as e:
                if "width mismatch" not in str(e):
                    raise
                return m.sample_rb(n, seed, batch_size=bs, threads=threads)  # run_batch restatement (SURVEY finding 2)
        kind = "reference"
    else:
        om = coracle.OracleModel.load(path)

        def run(n):
            return om.sample(n, seed)
        kind = "port"
        threads = 1
    n = 64 * threads
    run(n)  # warm-up (first cold run is slow)
    while True:
        t = time.perf_counter()
        run(n)
        dt = time.perf_counter() - t
        if dt > 0.5 or n >= (1 << 30):
            break
        n *= 4
    n = int(min(1 << 31, max(64, n * target_s / max(dt, 1e-6))))
    n = (n + 63) // 64 * 64
    t = time.perf_counter()
    run(n)
    dt = time.perf_counter() - t
    return n / dt, n, kind, dt, threads


def run_reference_arm(args, wl):
    rank, world, local = dist_env()
    if rank != 0:
        return
    path = os.path.join(ROOT, wl[0])
    threads = os.cpu_count() or 1
    steps = []
    kind = "reference"
    n = 0
    for i in range(args.warmup + args.steps):
        rate, n, kind, dt, used = reference_rate(path, args.ref_seconds, seed=1 + i, threads=threads)
        if i >= args.warmup:
            steps.append(rate)
    value = statistics.median(steps)
    line = {"impl": "reference", "metric": "detector_shots_per_sec", "value": value, "unit": "shots/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": n / value * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32+f64",
            "data": "synthetic circuit (in-repo generator), compiled by the reference front-end",
            "config": {"workload": args.workload, "baseline_config": wl[1], "description": wl[2],
                       "shots_per_step": n},
            "cpu_baseline": {"value": value, "unit": "shots/s", "cores": used, "kind": kind,
                             "sample": f"{n} shots of {args.workload} per step, sample_detectors force_dense, "
                                       f"batch 65536, {used} threads ({cpu_model()})"},
            "e2e": {"value": value, "unit": "shots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2604_01059_b200 as zx

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    path = os.path.join(ROOT, wl[0])
    cs = zx.CompiledSampler.load(path, device=local)
    info = cs.info
    shots = args.shots or wl[3]
    shots = (shots + 63) // 64 * 64
    words = shots // 64
    count_only = wl[4]
    nout = cs.num_outputs
    cols = None if count_only else torch.empty((nout, words), dtype=torch.int64, device=dev)
    counts = torch.zeros(nout, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    seed = 1

    def step(i):
        first = (i * world + rank) * shots  # disjoint global shot ranges
        cnt = counts.data_ptr() if (count_only or world > 1) else 0  # logical-error counts for the reduction
        cs.sample_device(seed, first, shots, 0 if cols is None else cols.data_ptr(), words, cnt, sptr)

    for i in range(args.warmup):
        step(i)
    cs.check_errors(sptr)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    counts.zero_()
    cs.kernel_timing(True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # evict L2 between timed steps (outside the events)
            evs[i][0].record(stream)
            step(args.warmup + i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    cs.check_errors(sptr)
    ktimes = cs.kernel_times()
    cs.kernel_timing(False)
    kernel_ms = [a.elapsed_time(b) for a, b in evs]
    t_local = sum(kernel_ms)
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = tt.item()
        dist.all_reduce(counts)  # the only collective: per-output flip counts
    else:
        t_max = t_local
    total_shots = shots * args.steps * world
    value = total_shots / (t_max / 1e3)
    ms_per_step = t_max / args.steps

    # ---- e2e through the C-ABI host entry (zxs_sample -> host columns)
    e2e_shots = min(shots, args.e2e_shots)
    host = torch.empty((nout, (e2e_shots + 63) // 64), dtype=torch.int64).pin_memory()
    hnp = host.numpy().view(np.uint64)
    for i in range(2):
        cs.sample_into(cs.mode, seed, i * e2e_shots, e2e_shots, hnp)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        cs.sample_into(cs.mode, seed, ((i * world) + rank) * e2e_shots, e2e_shots, hnp)
    e2e_local = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([e2e_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_local = tt.item()
    e2e_value = e2e_shots * args.steps * world / e2e_local

    # ---- roofline of the dominant kernel (DESIGN.md "Kernels and their
    # rooflines"), timed per launch with CUDA events on the launch stream.
    launches = sum(n for _, n in ktimes.values())
    if info["num_mono_components"]:
        # mono_kernel: one conflict-free 128 B shared-memory wavefront per
        # selector per warp (32 lanes x 32 shots); algorithmic bytes =
        # plane loads per 32-shot word x 4 B x words. Peak: the same LDS+XOR
        # op mix measured live (zxs_measure_smem_peak).
        kms, kn = ktimes["mono_kernel"]
        per_launch_s = kms / max(kn, 1) / 1e3
        algo = shots / 32 * info["num_mono_loads"] * 4
        achieved = algo / per_launch_s / 1e9
        peak = zx.measure_smem_peak(local) / 1e9
        roof = {"bound": "smem", "kernel": "mono_kernel", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": args.traffic_bytes,
                "basis": f"{info['num_mono_loads']} parameter-plane loads per 32-shot word per chain pass "
                         f"(4 B each, {info['num_mono_records']} records), {algo:.3e} B per launch",
                "peak_source": "measured live: zxs_measure_smem_peak (conflict-free LDS.32 + XOR, same op mix)",
                "kernel_ms_per_launch": per_launch_s * 1e3,
                "kernel_share": kms / max(sum(v for v, _ in ktimes.values()), 1e-9)}
    else:
        # shot_kernel: bound by the 32x32->64 integer multiplies of
        # Philox4x32-10 (IMAD.WIDE on the fmaheavy pipe). Algorithmic work =
        # Philox blocks per shot (mechanisms + autoregressive draws); peak =
        # the same Philox code with no other work, measured live.
        kms, kn = ktimes["shot_kernel"]
        per_launch_s = kms / max(kn, 1) / 1e3
        blocks_per_shot = info["philox_blocks_per_shot"]
        achieved = shots * blocks_per_shot / per_launch_s / 1e9
        peak = zx.measure_philox_peak(local) / 1e9
        roof = {"bound": "int", "kernel": "shot_kernel", "achieved": achieved, "peak": peak,
                "unit": "GPhilox-blocks/s", "frac": achieved / peak, "traffic": args.traffic_bytes,
                "basis": f"{blocks_per_shot} Philox4x32-10 blocks/shot ({info['num_mechanisms']} mechanisms + "
                         f"{blocks_per_shot - info['num_mechanisms']} autoregressive draws)",
                "peak_source": "measured live: zxs_measure_philox_peak (same Philox code, no other work); "
                               "integer-multiply (fmaheavy) bound",
                "kernel_ms_per_launch": per_launch_s * 1e3,
                "kernel_share": kms / max(sum(v for v, _ in ktimes.values()), 1e-9)}
    roof["hbm"] = {"bytes_per_step": int(nout * words * 8) if not count_only else int(nout * 8),
                   "achieved_gbs": (nout * words * 8 if not count_only else 0) / (ms_per_step / 1e3) / 1e9,
                   "peak_gbs": MEASURED_HBM_GBS}
    clocks = clk.summary()
    line = {
        "metric": "detector_shots_per_sec", "value": value, "unit": "shots/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32+f64",
        "data": "synthetic circuit (in-repo generator), compiled by the reference front-end; L2 flushed between steps",
        "config": {"workload": args.workload, "baseline_config": wl[1], "description": wl[2],
                   "shots_per_gpu_per_step": shots, "parallelism": f"shot-range dp{world}",
                   "count_only": count_only, "l2": "flushed (256 MiB write) between timed steps"},
        "e2e": {"value": e2e_value, "unit": "shots/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(nout * ((e2e_shots + 63) // 64) * 8), "shots_per_step": e2e_shots},
        "gpu_launches": launches,
        "kernels": {k: {"ms": v, "launches": n} for k, (v, n) in ktimes.items() if n},
        "roofline": roof,
        "clocks": clocks,
        "kernel_ms": kernel_ms if len(kernel_ms) <= 20 else None,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, n, kind, dt, used = reference_rate(path, args.cpu_seconds, seed=1, threads=os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": rate, "unit": "shots/s", "cores": used, "kind": kind,
                                "sample": f"{n} shots of {args.workload}, {dt:.1f}s, {cpu_model()}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--shots", type=int, default=0, help="shots per GPU per step (default: per workload)")
    ap.add_argument("--e2e-shots", type=int, default=1 << 24)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=3.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic-bytes", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture of this configuration")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
