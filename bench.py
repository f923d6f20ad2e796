#!/usr/bin/env python3
"""Benchmark of the per-step effective-field + LLG hot path (BASELINE.json).

One "step" = Simulation<T>::step (sim.hpp:33-42): demag convolution (6 FFT
passes + tensor product), exchange + anisotropy + Zeeman, LLG right-hand
side, Euler update with |M| = Ms renormalisation and the max-torque
reduction, on a grid of BASELINE.json's configs.

Default workload (N=1): configs[3], the 512x512x64 thin film on which the
north-star roofline target is quoted (>= 60% of HBM roofline per LLG step);
fp32, cubic 2.5 nm cells, permalloy-like material with all four field terms
active.  Synthetic data: uniform (1,1,1)/sqrt(3) start.

Arms:
  python bench.py [--gpus N --steps K --warmup W]     this engine (libmagfd_b200.so)
  python bench.py --impl reference ...                 the reference CPU code (oracle/_ref)

Multi-GPU (torchrun, N>1): the z-slab decomposition over NCCL (strong scaling
of the one grid: each rank owns nz/N planes; two all-to-all transposes of the
x-spectrum per step + a one-plane M halo).  If the slab path cannot start on
any rank, every rank fails (no silent fallback).  See DESIGN.md section (e).

Both arms print the same `config` object (the grid the step runs on); the CPU
legs run the reference on the full grid with all host threads, plus a 1-thread
row.
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (nx, ny, nz, dx, dy, dz), BASELINE.json config string
    "film512": ((512, 512, 64, 2.5e-9, 2.5e-9, 2.5e-9), "thin film 512x512x64 cells (BASELINE configs[3])"),
    "sp4": ((128, 32, 1, 500e-9 / 128, 125e-9 / 32, 3e-9), "muMAG SP4 128x32x1 (configs[0])"),
    "sp4fine": ((512, 128, 4, 500e-9 / 512, 125e-9 / 128, 0.75e-9), "SP4 refined 512x128x4 (configs[1])"),
    "cube128": ((128, 128, 128, 2.5e-9, 2.5e-9, 2.5e-9), "permalloy cube 128^3 (configs[2])"),
    "film1024": ((1024, 1024, 128, 2.5e-9, 2.5e-9, 2.5e-9), "large film 1024x1024x128 (configs[4])"),
}
MATERIAL = dict(A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.02, easy_axis=(0.0, 0.0, 1.0))
H_EXT = (1e4, 0.0, 0.0)
DT = 1e-14
METRIC = "LLG cell-updates/s per step (N x steps/s) + % HBM roofline"
UNIT = "cell-updates/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def model_bytes_per_kernel(g, s):
    """Algorithmic HBM bytes of each pass (SURVEY.md section 8d, 5-pass model)."""
    nx, ny, nz = g[:3]
    N = nx * ny * nz
    P = lambda n: 1 << (2 * n - 1).bit_length()
    Px, Py, Pz = P(nx), P(ny), P(nz)
    Hx = Px // 2 + 1
    c = 2 * s
    k1 = 3 * N * s + 3 * Hx * ny * nz * c
    k2 = 3 * Hx * ny * nz * c + 3 * Hx * Py * nz * c
    k3 = 2 * (3 * Hx * Py * nz * c) + 6 * Hx * (Py // 2 + 1) * (Pz // 2 + 1) * s
    k4 = k2
    k5 = 3 * Hx * ny * nz * c + 6 * N * s
    return {"k_r2c_x": k1, "k_fft_y_fwd": k2, "k_fft_z_conv": k3, "k_fft_y_inv": k4, "k_c2r_x_llg": k5}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.idx = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                self.samples.append([v.strip() for v in line.split(",")])

        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx = float(s[1])
                for n, v in zip(names, s[3:7]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(ws, v):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------- CPU reference
def cpu_reference(steps, warmup, threads, grid, precision=32, budget_s=None, one_thread_steps=0):
    """Reference Simulation<T>::step (oracle/_ref, the unmodified reference code) on
    the host cores: setup on `threads` threads (timed separately), `warmup` steps,
    then the median of `steps` per-step wall times (the reference bench protocol,
    cli.cpp:95-117), stopping early once `budget_s` of stepping is spent.  With
    one_thread_steps > 0 the same state then steps on a 1-thread backend.
    Returns dict(value, ms, setup_s, steps, ms_1thread, steps_1thread)."""
    from oracle import oracle as O
    if not O.ref_available():
        raise RuntimeError("oracle/_ref/libmagfd_ref.so not built")
    import numpy as np
    spec = O.Spec(*grid, **MATERIAL, h_ext=H_EXT, dt=DT, parallel=True, threads=threads)
    t0 = time.perf_counter()
    r = O.Ref(spec, precision)
    n = spec.n
    r.set_m(np.full((3, n), 8e5 / 3 ** 0.5))
    setup = time.perf_counter() - t0

    def timed(k, budget):
        times = []
        for _ in range(k):
            t1 = time.perf_counter()
            r.step(1)
            times.append(time.perf_counter() - t1)
            if budget and sum(times) > budget:
                break
        return times

    r.step(warmup)
    times = timed(steps, budget_s)
    ms = statistics.median(times) * 1e3
    out = {"value": n / (ms / 1e3), "ms": ms, "setup_s": setup, "steps": len(times),
           "ms_1thread": None, "steps_1thread": 0}
    if one_thread_steps > 0:
        r.set_step_threads(1)
        t1 = timed(one_thread_steps, None)
        out["ms_1thread"] = statistics.median(t1) * 1e3
        out["steps_1thread"] = len(t1)
    return out


def config_of(workload, prec):
    """The `config` object both arms print (identical for the same grid / precision)."""
    g = WORKLOADS[workload][0]
    dt = "f32" if prec == 32 else "f64"
    return {"workload": WORKLOADS[workload][1], "grid": list(g[:3]), "cell_m": list(g[3:]),
            "precision": dt, "terms": "demag+exchange+anisotropy+zeeman",
            "material": "Ms 8e5, A 1.3e-11, Ku 4e4 (z), H_ext (1e4,0,0) A/m, alpha 0.02, dt 1e-14 s"}


def run_reference_arm(args, ws, rank):
    """The reference's own CPU implementation on the same grid as our arm (the full
    BASELINE grid, all host threads).  A step takes seconds at the film sizes, so
    the warm-up is capped at 3 steps (the reference bench's own count,
    cli.cpp:95-99) and the timed steps stop after a 150 s budget."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    g = WORKLOADS[args.workload][0]
    warm = min(args.warmup, 3)
    try:
        r = cpu_reference(args.steps, warm, threads, g, args.precision, budget_s=150)
    except Exception as e:  # reference not built on this box
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return
    ct = "float" if args.precision == 32 else "double"
    dt = "f32" if args.precision == 32 else "f64"
    desc = (f"reference Simulation<{ct}>::step (oracle/_ref, built from /root/reference/proj with its "
            f"Release flags) on the full {g[0]}x{g[1]}x{g[2]} grid, {threads} host threads; {warm} warm-up + "
            f"median of {r['steps']} steps; setup {r['setup_s']:.1f}s excluded")
    out = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": r["steps"], "warmup": warm, "ms_per_step": r["ms"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic (uniform (1,1,1)/sqrt3 start)",
        "config": config_of(args.workload, args.precision),
        "execution": f"CPU, {threads} host threads (reference Backend parallel)",
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "reference", "sample": desc,
                         "setup_s": r["setup_s"]},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def cpu_sample_grid(g):
    """Bounded CPU sample: shrink x and y by 2 until <= 2.1M cells (keeps nz, cell size)."""
    nx, ny, nz = g[:3]
    while nx * ny * nz > 2_100_000 and nx > 8 and ny > 8:
        nx //= 2
        ny //= 2
    return (nx, ny, nz) + tuple(g[3:])


# --------------------------------------------------------------------- ours
def run_ours(args, ws, rank, local):
    import numpy as np
    import torch

    import paper_1406_7459_b200 as E

    torch.cuda.set_device(local)
    g = WORKLOADS[args.workload][0]
    prec = args.precision
    s = 4 if prec == 32 else 8
    grid = E.Grid(*g)
    mk = dict(precision=prec, device=local, init_direction=(3 ** -0.5,) * 3)
    mode = "1 GPU"
    if ws > 1:
        # z-slab decomposition over NCCL (strong scaling of one grid).  Every rank
        # learns whether all ranks started; any failure stops all of them.
        import torch.distributed as dist
        box = [E.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        sim, err = None, None
        try:
            sim = E.Simulation(grid, E.Material(**MATERIAL), E.FieldConfig(True, True, True, True, H_EXT),
                               E.StepperConfig(dt=DT), world=ws, rank=rank, nccl_id=box[0], **mk)
        except Exception as e:   # pragma: no cover - multi-GPU only
            err = e
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            raise RuntimeError(f"z-slab engine failed to start on rank {rank}: {err}" if err else
                               "z-slab engine failed to start on another rank")
        mode = f"z-slab x{ws} (NCCL all-to-all + halo over NVLink)"
    else:
        sim = E.Simulation(grid, E.Material(**MATERIAL), E.FieldConfig(True, True, True, True, H_EXT),
                           E.StepperConfig(dt=DT), **mk)
    stream = torch.cuda.ExternalStream(sim.stream_handle(), device=torch.device("cuda", local))
    ncell = grid.cell_count                       # global cells of the grid
    slab_cells = sim.n                            # cells this rank owns
    replicas = 1

    # warm-up (graph capture + clocks ramp), then capture the timed run's graphs
    # so no capture / instantiation falls inside the timed region
    sim.step_async(args.warmup)
    sim.sync()
    launches = sim.prepare_async(args.steps)   # kernel nodes of the timed graphs

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sim.step_async(args.steps)
    e1.record(stream)
    e1.synchronize()
    sim.sync()
    torch.cuda.synchronize()
    barrier(ws)
    clk = clocks.stop()
    ms_total = allmax(ws, e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    value = replicas * ncell * args.steps / (ms_total / 1e3)

    # per-kernel device time (events between passes, real steps on the same stream)
    reps = max(5, min(20, args.steps))
    acc = np.zeros(7)
    for _ in range(reps):
        acc += sim.step_timing()
    per = acc / reps
    names = ["k_r2c_x", "k_fft_y_fwd", "k_fft_z_conv", "k_fft_y_inv", "k_c2r_x_llg"]
    per_kernel_ms = dict(zip(names, per[:5]))
    mb = model_bytes_per_kernel(g, s)
    if replicas == 1 and ws > 1:                  # per-rank share of the slab decomposition
        mb = {k: v / ws for k, v in mb.items()}
    top = max(per_kernel_ms, key=per_kernel_ms.get)
    peak, peak_src = peaks()
    achieved = mb[top] / (per_kernel_ms[top] / 1e3) / 1e9
    step_bytes = sum(mb.values())

    # e2e through the public API with pinned host buffers, every step: the host->device
    # copy of that step's input state M (mfd_stage_m, on a copy stream, overlapping the
    # previous step), the step (mfd_step_async) and the device->host read of its result
    # (mfd_sync_torque).  The serial form (mfd_set_m + mfd_step, no overlap) is kept
    # beside it as e2e_serial.
    e2e_steps = max(3, min(args.steps, 20))
    tdt = torch.float32 if prec == 32 else torch.float64
    hosts = [torch.empty((3, slab_cells), dtype=tdt).pin_memory().numpy() for _ in range(2)]
    cur_m = sim.get_m(dtype=np.float32 if prec == 32 else np.float64)
    for h in hosts:
        h[:] = cur_m
    sim.set_m(hosts[0])
    sim.step(1)                          # captures the 1-step graph outside the timed loops
    sim.stage_m(hosts[1])                # allocates the staging buffers / copy stream
    sim.step_async(1)
    sim.sync_torque()
    barrier(ws)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        sim.set_m(hosts[0])
        torque = sim.step(1)
    t_serial = allmax(ws, time.perf_counter() - t0)
    barrier(ws)
    t0 = time.perf_counter()
    sim.stage_m(hosts[0])
    for i in range(e2e_steps):
        sim.step_async(1)
        if i + 1 < e2e_steps:
            sim.stage_m(hosts[(i + 1) % 2])
        torque = sim.sync_torque()
    t_e2e = allmax(ws, time.perf_counter() - t0)
    e2e_value = replicas * ncell * e2e_steps / t_e2e
    e2e_serial = replicas * ncell * e2e_steps / t_serial

    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:   # per launch, keyed by workload and precision (one ncu --set full capture each)
            traffic = json.load(open(tp)).get(args.workload, {}).get("f32" if prec == 32 else "f64", {}).get(top)
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and ws == 1 and not args.skip_cpu:
        ct = "float" if prec == 32 else "double"
        try:
            threads = os.cpu_count() or 1
            r = cpu_reference(3, 1, threads, g, prec, budget_s=60, one_thread_steps=1)
            cpu = {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"reference Simulation<{ct}>::step (oracle/_ref) on the full {g[0]}x{g[1]}x{g[2]} grid, "
                             f"same material/cell size/terms, {threads} host threads: 1 warm-up + median of "
                             f"{r['steps']} steps ({r['ms']:.0f} ms/step); setup {r['setup_s']:.1f}s excluded",
                   "ms_per_step": r["ms"], "setup_s": r["setup_s"],
                   "one_thread": {"value": ncell / (r["ms_1thread"] / 1e3), "ms_per_step": r["ms_1thread"],
                                  "cores": 1, "steps": r["steps_1thread"]}}
            if args.workload == "film512":   # round-1 comparison point, kept as an extra field
                s2 = cpu_sample_grid(g)
                r2 = cpu_reference(3, 1, threads, s2, prec, budget_s=10)
                cpu["sample_128x128x64"] = {"value": r2["value"], "ms_per_step": r2["ms"], "grid": list(s2[:3])}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None,
            "dtype": "f32" if prec == 32 else "f64",
            "data": "synthetic (uniform (1,1,1)/sqrt3 start)",
            "config": config_of(args.workload, prec),
            "execution": mode,
            "l2": "working set > 126 MB L2 (no flush needed)" if step_bytes > 4e8 else
                  "working set fits L2 (inputs not flushed)",
            "timed_region": "graphs captured before the timed region (prepare_async); per-pass times from "
                            "event-record nodes of a captured one-step graph",
            "steps_per_s": 1e3 / ms_step,
            "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "model_bytes_per_launch": mb[top], "avg_launch_ms": per_kernel_ms[top]},
            "step_roofline": {"model_bytes_per_step": step_bytes, "achieved_GBps": step_bytes / (ms_step / 1e3) / 1e9,
                              "frac": step_bytes / (ms_step / 1e3) / 1e9 / peak},
            "per_kernel_ms": per_kernel_ms,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 3 * slab_cells * s, "d2h_bytes_per_step": 8,
                    "how": "per step: the step's input M from pinned host memory (C ABI mfd_stage_m, H2D on a copy "
                           "stream overlapping the previous step) + mfd_step_async + mfd_sync_torque (the step's "
                           "torque read back to the host)",
                    "serial": {"value": e2e_serial, "how": "per step: mfd_set_m (synchronous H2D) + mfd_step"}},
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="film512")
    ap.add_argument("--precision", type=int, choices=[32, 64], default=32)
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
