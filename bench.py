#!/usr/bin/env python
"""Benchmark of the UltraGauss training hot path on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Metric: fwd+bwd slices/s at config C3 -- 1M Gaussians (fixed init cloud,
init_cloud(seed=0, l_init U[0.85,1.05)) over the 160^3 shells phantom), 256x256
slices @0.375 mm at random poses.  A step is one full training step over a
batch of B slices per GPU: ugs_bin (phase 1 + tile sort) -> forward -> L1+SSIM
loss -> backward -> [NCCL all-reduce] -> grad stats -> Adam.  `value` is the
whole-job rate (B * N * K slices / max-over-ranks device time), inputs resident
in HBM; `e2e` repeats it with every step's targets copied from pinned host
memory and the loss read back.  `--impl reference` times the reference's CPU
path (the oracle port of echosplat; the Python reference cannot travel to
the GPU host) on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "slices/sec fwd+bwd (1M Gaussians, 256x256)"
UNIT = "slices/s"
# algorithmic work per (Gaussian, pixel) pair: operator
# counts of the reference kernels (_kernels.py:38-47 forward, :73-101 backward)
FLOP_FWD_PER_PAIR = 28
FLOP_BWD_PER_PAIR = 73


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=16, help="slices per GPU per step")
    ap.add_argument("--n-gaussians", type=int, default=1_000_000)
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--spacing", type=float, default=0.375)
    ap.add_argument("--n-slices", type=int, default=256, help="dataset size")
    ap.add_argument("--cpu-sample", type=int, default=48,
                    help="slices in the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tts", action="store_true",
                    help="skip the time-to-0.99-SSIM run (C2, N=1 only)")
    ap.add_argument("--tts-budget", type=float, default=120.0)
    ap.add_argument("--tts-runs", type=int, default=3)
    return ap.parse_args()


def workload_desc(a):
    return (f"C3: {a.n_gaussians} Gaussians (init_cloud seed 0, l_init U[0.85,1.05), "
            f"means U(+-48 mm)), {a.size}x{a.size} @{a.spacing} mm random-pose slices "
            f"(uniform rotation, t~U(+-12 mm)^3) of the 160^3 @0.6 mm shells phantom")


def make_phantom_and_specs(a):
    from paper_2505_05643_b200.volume import make_phantom
    from paper_2505_05643_b200.dataset import random_pose_specs
    vol = make_phantom("shells", 160, 0.6, seed=1)
    specs = random_pose_specs(a.n_slices, a.size, a.size, a.spacing, seed=0,
                              translate=12.0)
    return vol, specs


def train_config(a):
    from paper_2505_05643_b200.trainer import TrainConfig
    # scene-scale hyper-parameters (ref tests/test_acceptance.py:40-46)
    return TrainConfig(n_gaussians=a.n_gaussians, iterations=10000, seed=0,
                       l_init_low=0.85, l_init_high=1.05, lr_means_start=0.016,
                       lr_means_final=1.6e-4, lr_general_final=0.005,
                       heuristic_interval=0, batch=a.batch)


_SAMPLER = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
bus, period = sys.argv[1], float(sys.argv[2])
try:
    h = nv.nvmlDeviceGetHandleByPciBusId(bus)
except Exception:
    h = nv.nvmlDeviceGetHandleByIndex(0)
print("max", nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM), flush=True)
while True:
    t = time.monotonic()
    print(t, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
          nv.nvmlDeviceGetCurrentClocksEventReasons(h), flush=True)
    time.sleep(period)
"""


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.  A child
    process polls NVML (the library nvidia-smi reads) every `period` seconds
    and prints monotonic-clock timestamped samples; it is started before the
    warm-up (so its start-up cost is outside the timed region -- a
    `nvidia-smi -lms` child needs ~100 ms to start, longer than a 50-step
    timed region), `mark(t0, t1)` names the timed window and `stop()`
    summarises the samples inside it.  A separate process keeps the poll
    off this process's GIL."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("hw_power_brake_slowdown", 0x80),
               ("sw_power_cap", 0x4))

    def __init__(self, device=0, period=0.002):
        self.device = device
        self.period = period
        self.proc = None
        self.window = None
        self.err = None

    def start(self):
        import subprocess
        try:
            import torch
            p = torch.cuda.get_device_properties(self.device)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        except Exception:
            bus = "none"
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, bus, str(self.period)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            import atexit
            atexit.register(self._kill)     # never outlive the bench
            first = self.proc.stdout.readline().split()   # blocks until NVML is up
            self.sm_max = float(first[1])
        except Exception as e:  # pragma: no cover - no NVML
            self.err = f"nvml sampler unavailable: {e}"
            if self.proc is not None:
                self.proc.kill()
            self.proc = None

    def _kill(self):
        if self.proc is not None and self.proc.poll() is None:
            self.proc.kill()

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "not sampled"],
                    "samples": 0}
        time.sleep(2 * self.period)
        self.proc.terminate()
        out, _ = self.proc.communicate()
        rows = []
        for line in out.splitlines():
            f = line.split()
            try:
                rows.append((float(f[0]), float(f[1]), int(f[2])))
            except (ValueError, IndexError):
                continue
        scope = "all"
        if self.window is not None:
            inside = [r for r in rows if self.window[0] <= r[0] <= self.window[1]]
            if inside:
                rows, scope = inside, "timed"
        reasons = sorted({name for _, _, rs in rows for name, bit in self.REASONS if rs & bit})
        sm = [r[1] for r in rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.sm_max,
                "reasons": reasons, "samples": len(sm), "window": scope, "source": "nvml"}


# ------------------------------------------------------------------ CPU ---

def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:  # pragma: no cover
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference_rate(a, vol, specs, n_slices, cfg, warmup=1, workers=None):
    """The reference's per-iteration path (oracle port, all host cores):
    rasterize -> loss -> backward -> adam_step per slice.  Returns
    (slices/s, seconds, cores)."""
    from oracle import oracle as O
    from paper_2505_05643_b200.volume import sample_slice
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import cases
    cl = cases.uniform_cloud(cfg.seed, a.n_gaussians, vol.world_bounds(),
                             cfg.l_init_low, cfg.l_init_high)
    params = dict(cl)
    m = {k: np.zeros_like(params[k]) for k in O.GROUPS}
    v = {k: np.zeros_like(params[k]) for k in O.GROUPS}
    m["bg"] = np.zeros(2, np.float32)
    v["bg"] = np.zeros(2, np.float32)
    cores = workers or cpu_cores()
    targets = [sample_slice(vol, specs[i]).pixels for i in range(n_slices + warmup)]
    consts = [O.slice_constants(s.pose.rotation, s.pose.translation, s.width, s.height,
                                s.spacing, cfg.p_mass) for s in specs[:n_slices + warmup]]
    t = 0
    t0 = None
    init = {k: np.array(params[k], copy=True) for k in O.GROUPS}
    for i in range(n_slices + warmup):
        if i == warmup:
            t0 = time.perf_counter()
        t += 1
        # same fixed-cloud protocol as the GPU arm: every iteration starts
        # from the C3 init cloud, the copy counted in the time
        for k in O.GROUPS:
            params[k][...] = init[k]
        params["bg_intensity_raw"], params["bg_opacity_raw"] = 0.0, -4.0
        lr_g = O.general_lr(cfg.lr_general, cfg.lr_general_final, cfg.iterations, t)
        lrs = {"means": O.mean_lr(cfg.lr_means_start, cfg.lr_means_final, cfg.iterations, t),
               "l_raw": lr_g, "intensity_raw": lr_g, "opacity_raw": lr_g, "bg": lr_g}
        O.train_iteration(params, m, v, t, consts[i], targets[i], cfg.ssim_loss_weight,
                          lrs, cfg.p_mass, workers=cores)
    dt = time.perf_counter() - t0
    return n_slices / dt, dt, cores


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    vol, specs = make_phantom_and_specs(a)
    cfg = train_config(a)
    rate, dt, cores = cpu_reference_rate(a, vol, specs, a.steps, cfg, warmup=a.warmup)
    sample = (f"{a.steps} timed + {a.warmup} warm-up iterations, 1 slice each "
              f"(rasterize->loss->backward->adam_step from the fixed C3 init cloud, "
              f"workers={cores})")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1000.0 * dt / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 pair math / f32 accum",
            "data": "synthetic", "config": {"workload": workload_desc(a),
                                            "batch_per_step": 1,
                                            "implementation": "oracle port of echosplat (C + numpy), host CPU"},
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU ---

def fp32_peak_tflops(torch):
    from paper_2505_05643_b200 import _lib
    L = _lib.lib()
    out = torch.zeros(1, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sms * 8, 20000
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.ugs_fp32_peak_probe(out.data_ptr(), blocks, iters, st), "probe")
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = max(best, blocks * 256.0 * iters * 16 / (ms * 1e-3) / 1e12)
    return best


def run_ours(a):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # UGS_BENCH_ONE_DEVICE=1 (tests only): every rank on cuda:0 over gloo, to
    # exercise the N > 1 code path on a one-GPU box (NCCL refuses that)
    one_dev = os.environ.get("UGS_BENCH_ONE_DEVICE", "0") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        if one_dev:
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl",
                                                 device_id=torch.device("cuda", local))
    import paper_2505_05643_b200 as ug
    from paper_2505_05643_b200 import _lib
    from paper_2505_05643_b200.trainer import TrainEngine

    vol, specs = make_phantom_and_specs(a)
    targets = ug.sample_slices(vol, specs, device="cuda")
    cfg = train_config(a)
    cloud = ug.init_cloud(cfg, vol.world_bounds(), device="cuda")
    eng = TrainEngine(cloud, cfg, specs, targets, world, rank, pg)
    B = a.batch
    order_rng = np.random.default_rng(1234)
    order = order_rng.permutation(len(specs))
    cursor = [0]

    def next_batch():
        picks = []
        for _ in range(B * world):
            if cursor[0] >= len(order):
                cursor[0] = 0
            picks.append(int(order[cursor[0]]))
            cursor[0] += 1
        return picks[rank * B:(rank + 1) * B]

    it = [0]
    # SURVEY 8(d) C3 fixes the cloud distribution (P ~ 25-40M pairs/slice);
    # training would otherwise grow the footprints step by step (lr 0.05 on
    # l_raw).  Every step therefore starts from the fixed init cloud: a device
    # copy of the 44 B/Gaussian parameters, paid inside the timed region.
    init = [t.clone() for t in (cloud.means, cloud.l_raw, cloud.intensity_raw,
                                cloud.opacity_raw, cloud.bg_raw)]

    # the step's loss goes device -> pinned host memory asynchronously; the
    # host reads (and checks) step i's loss while step i+1 runs, so no step
    # waits for its own loss (the reference aborts on a non-finite loss,
    # trainer.py:392-396; here a non-finite loss fails the bench)
    loss_host = torch.empty(1 << 12, dtype=torch.float64).pin_memory()
    loss_ev = [None] * loss_host.numel()

    def read_loss(i):
        if i < 0 or loss_ev[i % len(loss_ev)] is None:
            return None
        loss_ev[i % len(loss_ev)].synchronize()
        v = float(loss_host[i % len(loss_ev)])
        if not np.isfinite(v):
            raise RuntimeError(f"non-finite loss at step {i}")
        return v

    pending = [None]      # (step number, device loss) of the last launched step

    def flush_loss():
        """Queue the D2H copy of the last launched step's loss.  Called once
        that step is final: the engine settles a step (harvests its sync-free
        binning counts, re-issues it if it overflowed the plan) at the start
        of the next one, or in settle()."""
        if pending[0] is None:
            return
        i, lt = pending[0]
        k = i % len(loss_ev)
        loss_host[k].copy_(lt, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        loss_ev[k] = ev
        pending[0] = None

    def step(targets_batch=None, idx=None):
        it[0] += 1
        c = eng.cloud
        # one multi-tensor copy kernel (5 separate DtoD memcpys cost ~36 us)
        torch._foreach_copy_([c.means, c.l_raw, c.intensity_raw, c.opacity_raw, c.bg_raw],
                             init)
        lt = eng.step(idx if idx is not None else next_batch(), it[0],
                      targets_batch=targets_batch, check_finite=False)
        flush_loss()                      # the previous step (final now)
        pending[0] = (it[0], lt)
        return read_loss(it[0] - 2)       # two back: never waits on a running step

    def finish():
        eng.settle()
        flush_loss()
        read_loss(it[0] - 1)
        read_loss(it[0])

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(a.warmup):
        step()
    finish()
    # ---- timed region: device-resident inputs, no instrumentation ----
    eng.pairs_total = 0
    barrier()
    torch.cuda.synchronize()
    t_host0 = time.monotonic()
    l0 = _lib.lib().ugs_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")      # ncu --nvtx-include "timed/"
    e0.record()
    for _ in range(a.steps):
        step()
    finish()
    e1.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    sampler.mark(t_host0, time.monotonic())
    launches = _lib.lib().ugs_launch_count() - l0
    clocks = sampler.stop()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    pairs_per_step = eng.pairs_total / a.steps
    # ---- the same K steps again with per-stage CUDA events on the launch
    # stream (the roofline's kernel times); kept out of `value` because the
    # event records add host latency after the binning sync (~3 %) ----
    eng.renderer.set_timing(True)
    eng.renderer.timings(reset=True)
    eng.profile = True
    eng.event_times(reset=True)
    barrier()
    torch.cuda.synchronize()
    for _ in range(a.steps):
        step()
    finish()
    torch.cuda.synchronize()
    stage = eng.renderer.timings()
    extra = eng.event_times()
    eng.profile = False
    eng.renderer.set_timing(False)
    value = B * world * a.steps / (ms * 1e-3)

    # ---- e2e: host-pinned targets copied every step, loss read back ----
    e2e = None
    if not a.no_e2e:
        host_t = targets.cpu().pin_memory()
        # the step's target slices go straight from the pinned host dataset to
        # a double-buffered device batch, one H2D copy per slice on a copy
        # stream, so step i+1's upload overlaps step i's compute (a device
        # buffer is refilled only after the step that read it)
        dev_t = [torch.empty((B, a.size, a.size), dtype=torch.float32, device="cuda")
                 for _ in range(2)]
        copy_stream = torch.cuda.Stream()
        st_ev, used_ev = [None, None], [None, None]
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        f0.record()
        for i in range(a.steps):
            idx = next_batch()
            b = i & 1
            with torch.cuda.stream(copy_stream):
                if used_ev[b] is not None:
                    copy_stream.wait_event(used_ev[b])
                for j, sl in enumerate(idx):
                    dev_t[b][j].copy_(host_t[sl], non_blocking=True)
                st_ev[b] = torch.cuda.Event()
                st_ev[b].record(copy_stream)
            torch.cuda.current_stream().wait_event(st_ev[b])
            r0 = eng.reissued
            step(targets_batch=dev_t[b], idx=idx)     # + D2H read of an earlier loss
            # buffer b is read by this step -- and buffer 1-b again if the
            # previous step was re-issued inside this call (binning overflow)
            for q in ((b, 1 - b) if eng.reissued != r0 else (b,)):
                used_ev[q] = torch.cuda.Event()
                used_ev[q].record()
        finish()                                   # ... and of the last one
        f1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        ms_e2e = max_over_ranks(max(f0.elapsed_time(f1), wall * 1e3))
        h2d = B * a.size * a.size * 4 + B * 144 + 16 * B
        d2h = 8 + 24 * B
        e2e = {"value": B * world * a.steps / (ms_e2e * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    # ---- roofline (dominant kernel) ----
    peak_fp32 = fp32_peak_tflops(torch)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # per step (a stage may launch more than once per step)
    stage_ms = {k: v[0] / a.steps for k, v in stage.items()}
    stage_ms.update({k: v[0] / a.steps for k, v in extra.items()})
    dom = max(("forward", "backward"), key=lambda k: stage_ms.get(k, 0.0))
    flop_pp = FLOP_BWD_PER_PAIR if dom == "backward" else FLOP_FWD_PER_PAIR
    achieved = flop_pp * pairs_per_step / (stage_ms[dom] * 1e-3) / 1e12
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(dom + "_kernel_dram_bytes")
    except (OSError, ValueError):
        pass
    # the dominant kernel's own pipe view from the newest committed ncu
    # capture (frac is on the reference's operator count; see the note)
    executed = None
    try:
        import glob
        nf = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_full_r*.json")))[-1]
        for k in json.load(open(nf))["kernels"]:
            if k["kernel"] == dom + "_kernel":
                executed = {
                    "source": os.path.relpath(nf, ROOT),
                    "issue_active_pct": float(k["smsp__issue_active.avg.pct_of_peak_sustained_active"].split()[0]),
                    "fma_pipe_inst_pct": float(k["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"].split()[0]),
                    "xu_pipe_inst_pct": float(k["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"].split()[0]),
                    "warp_instructions": float(k["smsp__inst_executed.sum"].split()[0])}
    except (OSError, ValueError, IndexError, KeyError):
        pass
    n = eng.cloud.n
    # parameter update (update_gather_kernel): N=1 fuses accumulate + stats +
    # Adam -- reads params 44 B + m, v 96 B and writes them back (280 B per
    # Gaussian) plus 48 B per record gradient row; N>1 adds the dense AoS-12
    # gradient row write (48 B) and a separate Adam (ugs_adam_step, +96 B)
    m_per_step = float(np.sum(eng.renderer.m)) if hasattr(eng.renderer, "m") else 0.0
    upd_stage = "update" if world == 1 else "adam"
    upd_bytes = (280 * n + 48 * m_per_step) if world == 1 else (376 + 48) * n + 48 * m_per_step
    upd_ms = stage_ms.get(upd_stage, float("nan"))

    def tflops(fpp, k):
        return fpp * pairs_per_step / (stage_ms.get(k, float("nan")) * 1e-3) / 1e12

    roof_stages = {
        "forward": {"flops": FLOP_FWD_PER_PAIR * pairs_per_step, "ms": stage_ms.get("forward"),
                    "tflops": tflops(FLOP_FWD_PER_PAIR, "forward"),
                    "frac": tflops(FLOP_FWD_PER_PAIR, "forward") / peak_fp32},
        "backward": {"flops": FLOP_BWD_PER_PAIR * pairs_per_step, "ms": stage_ms.get("backward"),
                     "tflops": tflops(FLOP_BWD_PER_PAIR, "backward"),
                     "frac": tflops(FLOP_BWD_PER_PAIR, "backward") / peak_fp32},
        "update": {"stage": upd_stage, "bytes": upd_bytes, "ms": upd_ms,
                   "gbs": upd_bytes / (upd_ms * 1e-3) / 1e9,
                   "frac_of_hbm": upd_bytes / (upd_ms * 1e-3) / 1e9 / hbm_peak},
    }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (160^3 shells phantom, random-pose GT slices, random-init cloud)",
        "config": {"workload": workload_desc(a), "n_gaussians": a.n_gaussians,
                   "slice": [a.size, a.size], "batch_per_gpu": B, "global_batch": B * world,
                   "parallelism": f"dp{world}" + (
                       "" if world == 1 else
                       " (fused reduce-scatter+Adam+all-gather over NVLink peer memory)"
                       if eng.peer else " (NCCL all-reduce + replicated Adam)"),
                   "step": "param reset to the fixed C3 cloud (device copy)+ugs_bin+forward+"
                           "loss(L1+0.2*SSIM, f64)+backward+"
                           + ("" if world == 1 else "peer update (reduce-scatter+Adam+all-gather)+"
                              if eng.peer else "allreduce+") + "grad_stats+Adam",
                   "l2": "inputs larger than L2: params+Adam moments+grads = "
                         f"{(44 + 88 + 44) * n / 1e6:.0f} MB streamed per step",
                   "pairs_per_slice": pairs_per_step / B},
        "roofline": {"bound": "fp32", "kernel": dom + "_kernel", "achieved": achieved,
                     "peak": peak_fp32, "unit": "TFLOP/s", "frac": achieved / peak_fp32,
                     "traffic": traffic,
                     "traffic_source": "profiles/ncu_traffic.json: dram__bytes_read.sum + "
                                       "dram__bytes_write.sum of this kernel from one ncu "
                                       "--set full capture of the same command (not "
                                       "measurable inside an uninstrumented run)",
                     "note": f"algorithmic {flop_pp} FLOP/pair (reference operator count, "
                             "SURVEY 8d) x pairs per launch / CUDA-event launch time (stage "
                             "events on the launch stream, a second pass of the same K steps); "
                             "peak = FP32 FFMA probe measured in this run (no tensor cores: "
                             "not a dense contraction).  frac near or above 1 says the kernel "
                             "does fewer operations per pair than the reference's count "
                             "(plane-conditioned exponent: 2 packed FMAs + one ex2 per pixel "
                             "pair, moments instead of per-pair parameter chains); how busy "
                             "the SM actually is: `executed` (ncu, issue-bound with the FMA "
                             "and MUFU pipes co-saturated in the pixel loop)",
                     "executed": executed},
        "roofline_stages": roof_stages,
        "stage_ms_per_step": stage_ms,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not a.no_tts:
        # before the CPU legs: their host threads perturb a wall-clock
        # training measurement that follows them (2.86 s -> 3.1-4.0 s)
        # BASELINE metric part 2: time to 0.99 held-out SSIM (config C2, 1 GPU)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import time_to_ssim
        del eng
        torch.cuda.empty_cache()
        # training batch 48 (the fastest of 8..64 to 0.99 on C2, measured:
        # 8: 28.6 s, 16: 11.9 s, 32: ~5 s, 48: 4.0 s, 64: 5.2 s)
        # three runs, the median reported: a wall-clock training run here
        # carries the driver's allocation latency (the plan's buffers grow
        # ~20x in the first steps and cudaMalloc / cudaFree occasionally take
        # 100+ ms on these boxes): single runs scatter 2.9-4.0 s
        runs = [time_to_ssim.run(budget=a.tts_budget, batch=48, eval_every=10,
                                 log=lambda m: None) for _ in range(a.tts_runs)]
        reached = [x["reached_s"] for x in runs]
        order = sorted(range(len(runs)),
                       key=lambda j: float("inf") if reached[j] is None else reached[j])
        r = runs[order[len(runs) // 2]]
        line["time_to_ssim"] = {k: r[k] for k in ("target", "reached_s", "best_ssim",
                                                  "iterations", "slices_trained")}
        line["time_to_ssim"]["runs_reached_s"] = reached
        line["time_to_ssim"]["statistic"] = f"median of {len(runs)} runs"
        line["time_to_ssim"]["config"] = ("C2: 200k Gaussians, 160^3 shells phantom, "
                                          "256x256 @0.375 mm, 2048 train / 64 held-out "
                                          "random-pose slices, batch 48, held-out SSIM "
                                          "every 10 steps (not timed), 1 GPU")
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            rate, dt, cores = cpu_reference_rate(a, vol, specs, a.cpu_sample, cfg, warmup=1)
            # the reference's sequential mode too (workers=1, its
            # deterministic default), on a smaller sample
            n1 = max(2, a.cpu_sample // 8)
            rate1, dt1, _ = cpu_reference_rate(a, vol, specs, n1, cfg, warmup=1, workers=1)
            line["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                "cpu_model": cpu_model(),
                "sample": f"{a.cpu_sample} slices of the same workload, one reference "
                          f"iteration each (rasterize->loss->backward->adam_step), "
                          f"{dt:.1f} s, workers={cores}",
                "workers_1": {"value": rate1, "unit": UNIT, "cores": 1,
                              "sample": f"{n1} slices, {dt1:.1f} s, workers=1"}}
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": cpu_cores(),
                                    "kind": "port", "sample": f"failed: {exc!r}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
