"""Benchmark of the LEGO B200 backend (contract: one JSON line on rank 0).

Headline workload (BASELINE.json metric on its config 2, the largest
single-GPU remap config): the LEGO dimension-permutation layout
``GroupBy([16384,16384]).OrderBy(Col(16384,16384))`` applied to a
16384 x 16384 bf16 matrix -- every logical element (i, j) moves from its
row-major position to ``apply(i, j) = j*16384 + i``.  One step = one remap
of one matrix per GPU (weak scaling: N GPUs remap N independent matrices,
no data-path collective).  ``value`` = algorithmic bytes moved by all ranks
(read + write, 2 x 512 MiB per matrix) / max-over-ranks device time.

The input (512 MiB) and output are 4x the 126 MB L2, so no flush is needed
between iterations.  The other BASELINE configs are reported under
``"kernels"`` (measured in the same run, not the headline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 16384
HEADLINE_DSL = "GroupBy([16384,16384]).OrderBy(Col(16384,16384))"
METRIC = "layout-remap GB/s (frac of HBM peak); LEGO-GEMM TFLOP/s; 1/2/4/8 GPU"
WORKLOAD = ("cfg2: LEGO transpose layout GroupBy([16384,16384]).OrderBy(Col(16384,16384)) "
            "remapping a 16384x16384 bf16 matrix (row-major -> layout), 1 matrix per GPU per step")


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return {"hbm": float(p["hbm_gbs"]), "bf16": float(p["bf16_tflops"]),
                "bf16_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


def traffic_table():
    """Per-launch DRAM bytes from the committed ncu --set full captures."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001 - clocks are best effort
            self._nv = None
        return self

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 and os.environ.get("LEGO_BENCH_SHARE_GPU") == "1":
        # test hook: every rank on cuda:0 with a gloo group, so the multi-rank
        # control flow (barriers, max over ranks, the JSON line) runs on a
        # one-GPU box; numbers from such a run are not a scaling measurement
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    elif world > 1:
        import torch.distributed as dist
        # communicator lines (rank count per communicator) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def self_launch(args) -> int:
    """``--gpus N`` without a torchrun environment: start N ranks of this
    script through torch.distributed.run on 127.0.0.1 (NCCL_DEBUG=INFO so
    the communicator lines show N ranks) and return their exit code.  Rank
    0's JSON line reaches stdout unchanged."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """Rendezvous only (gloo, CPU): each rank reports the world it joined.
    Lets CPU tests check the multi-rank launch without a GPU."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
        got = dist.get_world_size()
        import torch
        t = torch.tensor([1])
        dist.all_reduce(t)
        ranks = int(t.item())
        dist.destroy_process_group()
    else:
        got, ranks = 1, 1
    sys.stderr.write(f"rank {rank} world={got}\n")
    sys.stderr.flush()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": got, "ranks_joined": ranks,
                          "workload": args.workload}), flush=True)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(value, world):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_steps(fn, steps, warmup, world):
    """W warm-up steps, then EXACTLY K timed steps bracketed by barrier +
    synchronize; device time from CUDA events on the launching stream."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    stream = torch.cuda.current_stream()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(steps):
        fn()
    end.record(stream)
    end.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(start.elapsed_time(end), world)


def kernel_event_time(fn, iters):
    """Average duration of the dominant launch (events around each launch)."""
    import torch
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(iters)]
    for s, e in evs:
        s.record(stream)
        fn()
        e.record(stream)
    torch.cuda.synchronize()
    return sum(s.elapsed_time(e) for s, e in evs) / iters


# ---------------------------------------------------------------------------
# CPU side (oracle port; test infrastructure, timed as the baseline only)
# ---------------------------------------------------------------------------

class CpuRemapSample:
    """The C oracle port of the reference per-element remap, timed on this
    host's cores over a bounded sample of the headline workload: buffers
    built and the sample size calibrated once, then one timed sample per
    step."""

    def __init__(self):
        import numpy as np
        from oracle import oracle as O
        self.O = O
        # every host core (torchrun presets OMP_NUM_THREADS=1 for its workers)
        O.set_threads(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
        self.spec = O.parse(HEADLINE_DSL)
        self.n = N * N
        self.src = (np.arange(self.n, dtype=np.uint32) & 0xFFFF).astype(np.uint16)
        self.out = np.zeros(self.n, dtype=np.uint16)
        self.count = N

    def calibrate(self, target_seconds):
        probe = 1 << 22
        self.O.remap(self.src, None, self.spec, first=0, count=probe, out=self.out)   # threads, pages
        t0 = time.perf_counter()
        self.O.remap(self.src, None, self.spec, first=0, count=probe, out=self.out)
        dt = time.perf_counter() - t0
        count = int(min(self.n, max(N, probe * target_seconds / max(dt, 1e-9))))
        self.count = max(N, count - count % N)
        return self.count

    def run(self):
        t0 = time.perf_counter()
        self.O.remap(self.src, None, self.spec, first=0, count=self.count, out=self.out)
        dt = time.perf_counter() - t0
        gbs = 2 * 2 * self.count / dt / 1e9
        threads = self.O.threads()
        return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                "sample": f"{self.count} of {self.n} 16-bit elements ({self.count // N} rows; bf16 moved as "
                          f"uint16 bit patterns) of the headline remap, oracle/lego_oracle.c per-element apply "
                          f"(reference layout.py:313) with {threads} OpenMP threads, {dt:.2f} s"}


def cpu_remap_rate(target_seconds=10.0):
    """One calibrated sample of the CPU port (the GPU arm's cpu_baseline)."""
    sample = CpuRemapSample()
    sample.calibrate(target_seconds)
    return sample.run()


def reference_python_rate():
    """The reference package's own per-element Python path (BASELINE.md
    4(i)), timed in the build container where the reference exists
    (scripts/time_reference_python.py -> profiles/r02_reference_python.json);
    reported beside the C port, not re-measured here."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_reference_python.json")) as fh:
            d = json.load(fh)
        c2 = d["layouts"]["cfg2"]
        return {"elements_per_s": c2["elements_per_s"], "GB/s_equivalent": round(c2["elements_per_s"] * 4 / 1e9, 6),
                "cores": d["cores"], "cpu": d.get("lscpu_model", d.get("cpu")),
                "sample": f"{d['sample_points']} points of the headline layout, reference layout.apply per element "
                          "on multiprocessing.Pool(all cores), measured in the build container "
                          "(profiles/r02_reference_python.json)"}
    except (OSError, KeyError, ValueError):
        return None


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the whole run (W + K samples) targets about 90 s of CPU work
    sample = CpuRemapSample()
    sample.calibrate(max(0.05, 90.0 / max(1, args.warmup + args.steps)))
    rates = []
    base = None
    for k in range(args.warmup + args.steps):
        r = sample.run()
        if k >= args.warmup:
            rates.append(r["value"])
            base = r
    value = sum(rates) / len(rates)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(2 * 2 * N * N / (value * 1e9) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic", "config": {"workload": WORKLOAD, "per_gpu_matrices": 1},
            "cpu_baseline": {**base, "value": round(value, 3)},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

def run(args):
    import torch

    import paper_2505_08091_b200 as L
    from paper_2505_08091_b200 import kernels as K

    world, rank, local = dist_setup(args)
    pk = peaks()
    layout = L.parse_layout(HEADLINE_DSL)
    nbytes = N * N * 2
    g = torch.Generator(device="cuda").manual_seed(1 + rank)
    src = torch.randn(N, N, generator=g, device="cuda", dtype=torch.float32).to(torch.bfloat16)
    src = src.reshape(N * N)
    out = torch.empty_like(src)
    step = lambda: K.remap(src, None, layout, out=out)  # noqa: E731
    step()
    # correctness spot check of the timed path: out[j*N + i] == src[i*N + j]
    probe = torch.randint(0, N, (2, 4096), device="cuda")
    ok = torch.equal(out[probe[1] * N + probe[0]], src[probe[0] * N + probe[1]])
    launches0 = K.LAUNCHES[0]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        ms = time_steps(step, args.steps, args.warmup, world)
    launches = K.LAUNCHES[0] - launches0 - args.warmup
    ms_step = ms / args.steps
    value = world * 2 * nbytes / (ms_step * 1e-3) / 1e9
    # dominant kernel = the remap itself (one launch per step): its average
    # launch duration over the timed region is the step time; events around
    # each launch separately (serialised, adds the event gaps) reported beside it
    kms = ms_step
    kms_each = kernel_event_time(step, max(5, min(args.steps, 20)))
    achieved = 2 * nbytes / (kms * 1e-3) / 1e9
    tr = traffic_table().get("remap_transpose_bf16")
    # context: a plain device copy of the same 512 MiB on this box, same timing
    scratch = torch.empty_like(src)
    copy_ms = time_steps(lambda: scratch.copy_(src), 20, 3, 1) / 20
    copy_gbs = 2 * nbytes / (copy_ms * 1e-3) / 1e9
    del scratch
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm"], "unit": "GB/s",
                "frac": round(achieved / pk["hbm"], 4), "peak_source": pk["source"],
                "frac_of_8000": round(achieved / 8000.0, 4),
                "traffic": tr, "algorithmic_bytes_per_launch": 2 * nbytes,
                "launch_us": round(kms * 1e3, 2),
                "launch_us_event_bracketed": round(kms_each * 1e3, 2),
                "same_size_copy_gbs": round(copy_gbs, 1),
                "frac_of_same_size_copy": round(achieved / copy_gbs, 4)}

    # e2e: public API with pinned host buffers.  Every step copies its input
    # host->device, remaps, and copies the result device->host, as a three-
    # stage pipeline over three buffer sets: an H2D stream, the remap stream
    # and a D2H stream, ordered per step by events, so the two copy engines
    # stream continuously in both directions (PCIe is full duplex) while each
    # step's three operations stay ordered.  A buffer set is reused three
    # steps later, once the remap has read its input and the D2H its output.
    NB = 3
    host_in = [torch.empty(N * N, dtype=torch.bfloat16, pin_memory=True) for _ in range(NB)]
    host_out = [torch.empty(N * N, dtype=torch.bfloat16, pin_memory=True) for _ in range(NB)]
    for h in host_in:
        h.copy_(src)
    dev_in = [torch.empty_like(src) for _ in range(NB)]
    dev_out = [torch.empty_like(src) for _ in range(NB)]
    h2d_s, cmp_s, d2h_s = (torch.cuda.Stream() for _ in range(3))
    ev_in = [torch.cuda.Event() for _ in range(NB)]
    ev_c = [torch.cuda.Event() for _ in range(NB)]
    ev_out = [torch.cuda.Event() for _ in range(NB)]
    main = torch.cuda.current_stream()
    e2e_counter = [0]

    def e2e_step():
        k = e2e_counter[0]
        e2e_counter[0] += 1
        b = k % NB
        if k >= NB:
            h2d_s.wait_event(ev_c[b])                   # the remap of step k-NB has read dev_in[b]
        with torch.cuda.stream(h2d_s):
            dev_in[b].copy_(host_in[b], non_blocking=True)
        ev_in[b].record(h2d_s)
        cmp_s.wait_event(ev_in[b])
        if k >= NB:
            cmp_s.wait_event(ev_out[b])                 # the D2H of step k-NB has read dev_out[b]
        K.remap(dev_in[b], None, layout, out=dev_out[b], stream=cmp_s)
        ev_c[b].record(cmp_s)
        d2h_s.wait_stream(cmp_s)
        with torch.cuda.stream(d2h_s):
            host_out[b].copy_(dev_out[b], non_blocking=True)
        ev_out[b].record(d2h_s)

    e2e_steps = max(8, args.steps // 4)

    def e2e_run():
        for _ in range(e2e_steps):
            e2e_step()
        for s in (h2d_s, cmp_s, d2h_s):
            main.wait_stream(s)

    for s in (h2d_s, cmp_s, d2h_s):
        s.wait_stream(main)
    for _ in range(6):
        e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(main)
    for s in (h2d_s, cmp_s, d2h_s):
        s.wait_event(t0)
    e2e_run()
    t1.record(main)
    t1.synchronize()
    e2e_ms = max_over_ranks(t0.elapsed_time(t1), world) / e2e_steps
    # the whole last result, as it arrived in host memory, against the
    # device-timed path's output for the same input (bit-exact, all 2^28 elements)
    ok_e2e = torch.equal(host_out[(e2e_counter[0] - 1) % NB].cuda(), out)
    e2e_value = world * 2 * nbytes / (e2e_ms * 1e-3) / 1e9

    kernels = {}
    if not args.headline_only:
        kernels = other_kernels(args, pk, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_remap_rate()
        ref_py = reference_python_rate()
        if ref_py:
            cpu["reference_python"] = ref_py

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (randn bf16, seed 1+rank)",
            "config": {"workload": WORKLOAD, "per_gpu_matrices": 1,
                       "layout": HEADLINE_DSL, "elem_bytes": 2,
                       "l2": "no flush: 512 MiB input + 512 MiB output per GPU >> 126 MB L2",
                       "parallelism": f"weak: {world} independent matrices, no data-path collective",
                       "check": "ok" if ok else "MISMATCH"},
            "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 1), "unit": "GB/s", "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes, "steps": e2e_steps,
                    "check": "ok" if ok_e2e else "MISMATCH",
                    "note": "public API kernels.remap; per step H2D of the input from pinned host "
                            "memory, remap, D2H of the whole result; a three-stage event pipeline "
                            "(H2D stream, remap stream, D2H stream, three buffer sets) keeps both "
                            "copy directions busy (PCIe-bound)"},
            "gpu_launches": launches, "clocks": clocks.summary(), "kernels": kernels,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _pinned_e2e(world, h2d_pairs, d2h_pairs, compute, steps):
    """End-to-end device time per step of: H2D of the inputs from pinned host
    memory, the compute, D2H of the outputs, on the current stream."""
    import torch
    def one():
        for dev, host in h2d_pairs:
            dev.copy_(host, non_blocking=True)
        compute()
        for host, dev in d2h_pairs:
            host.copy_(dev, non_blocking=True)
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        one()
    t1.record()
    t1.synchronize()
    return max_over_ranks(t0.elapsed_time(t1), world) / steps


def run_gemm_b8(args):
    """cfg5 as BASELINE.json states it: a batch of 8 bf16 8192^3 GEMMs
    (C = A B^T, tcgen05), batch-sharded 8/N per GPU -- strong scaling, no
    data-path collective."""
    import torch

    from paper_2505_08091_b200 import kernels as K, shard
    world, rank, _local = dist_setup(args)
    pk = peaks()
    B, n = 8, 8192
    p = shard.ShardPlan(B, world, rank)
    a = torch.empty(p.count, n, n, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    for i in range(p.count):
        g = torch.Generator(device="cuda").manual_seed(5 + 2 * (p.start + i))
        a[i] = torch.randn(n, n, generator=g, device="cuda").to(torch.bfloat16)
        b[i] = torch.randn(n, n, generator=g, device="cuda").to(torch.bfloat16)
    c = torch.empty_like(a)
    step = lambda: K.gemm(a, b, out=c)  # noqa: E731
    step()
    ref = torch.matmul(a[0, :64].double(), b[0].double().T) if p.count else None
    rel = 0.0
    if ref is not None:
        rel = ((c[0, :64].double() - ref).abs() / ref.abs().clamp_min(1e-2 * ref.abs().max().item())).max().item()
    launches0 = K.LAUNCHES[0]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        ms = time_steps(step, args.steps, args.warmup, world)
    launches = K.LAUNCHES[0] - launches0 - args.warmup
    ms_step = ms / args.steps
    flops = 2 * n ** 3 * B
    value = flops / (ms_step * 1e-3) / 1e12
    per_gpu = 2 * n ** 3 * max(p.count, 1) / (ms_step * 1e-3) / 1e12
    ha = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
    hb = torch.empty(b.shape, dtype=b.dtype, pin_memory=True)
    hc = torch.empty(c.shape, dtype=c.dtype, pin_memory=True)
    ha.copy_(a)
    hb.copy_(b)
    e2e_ms = _pinned_e2e(world, [(a, ha), (b, hb)], [(hc, c)], step, max(3, args.steps // 4))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        xa = a[0, :256].float().cpu()
        xb = b[0].float().cpu()
        torch.set_num_threads(len(os.sched_getaffinity(0)))
        torch.matmul(xa[:16], xb.T)
        t0 = time.perf_counter()
        torch.matmul(xa, xb.T)
        dt = time.perf_counter() - t0
        cpu = {"value": round(2 * 256 * n * n / dt / 1e12, 4), "unit": "TFLOP/s", "cores": torch.get_num_threads(),
               "kind": "port", "sample": f"256 rows of one 8192^3 GEMM, torch CPU fp32 matmul (restatement; the "
                                         f"reference has no GEMM), {dt:.2f} s"}
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "TFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (randn bf16, seeds 5+2k)",
                "config": {"workload": "cfg5: batch of 8 bf16 8192x8192x8192 GEMMs (C = A B^T) on tcgen05, "
                                       "batch-sharded 8/N per GPU", "per_gpu_matrices": p.count,
                           "parallelism": f"strong: batch 8 split over {world} GPUs, no data-path collective",
                           "l2": "no flush: 384 MiB of operands per GEMM >> 126 MB L2",
                           "check_max_rel_64_rows": rel},
                "roofline": {"bound": "tensor", "achieved": round(per_gpu, 1), "peak": pk["bf16"],
                             "unit": "TFLOP/s", "frac": round(per_gpu / pk["bf16"], 4),
                             "frac_sustained": round(per_gpu / pk["bf16_sustained"], 4), "traffic": None,
                             "peak_source": pk["source"]},
                "cpu_baseline": cpu,
                "e2e": {"value": round(flops / (e2e_ms * 1e-3) / 1e12, 1), "unit": "TFLOP/s",
                        "h2d_bytes_per_step": 2 * a.numel() * 2, "d2h_bytes_per_step": c.numel() * 2},
                "gpu_launches": launches, "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_transpose_shard(args):
    """cfg2 on ONE matrix split over N GPUs: rank r holds rows
    [r*n/N, (r+1)*n/N) of the 16384^2 bf16 matrix and ends with its share of
    the Col layout, through shard.FusedTranspose (one routed register
    transpose per rank storing into the peers' symmetric-memory shards over
    NVLink) -- strong scaling, the exchange fused into the remap kernel."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2505_08091_b200 import kernels as K, shard
    world, rank, _local = dist_setup(args)
    if world == 1:                      # symmetric memory needs a process group, even of one rank
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0,
                                device_id=torch.device("cuda", 0))
    n = N
    R = n // world
    g = torch.Generator(device="cuda").manual_seed(1 + rank)
    rows = torch.randn(R, n, generator=g, device="cuda").to(torch.bfloat16)
    ft = shard.FusedTranspose(n, n, rows.dtype, rows.device)
    step = lambda: ft(rows)  # noqa: E731
    out = step()
    torch.cuda.synchronize()
    C = n // world
    ok = torch.equal(out[:, rank * R:(rank + 1) * R], rows[:, rank * C:(rank + 1) * C].T)
    launches0 = K.LAUNCHES[0]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        ms = time_steps(step, args.steps, args.warmup, world)
    launches = K.LAUNCHES[0] - launches0 - args.warmup
    ms_step = ms / args.steps
    nbytes = 2 * n * n * 2
    value = nbytes / (ms_step * 1e-3) / 1e9
    pk = peaks()
    per_gpu = nbytes / world / (ms_step * 1e-3) / 1e9
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (randn bf16)",
                "config": {"workload": "cfg2 on one 16384x16384 bf16 matrix row-sharded over N GPUs -> Col layout "
                                       "(shard.FusedTranspose: routed register transpose into NVLink peer shards)",
                           "layout": HEADLINE_DSL, "check_own_block": "ok" if ok else "MISMATCH",
                           "parallelism": f"strong: {world} row shards, exchange fused into the remap kernel"},
                "roofline": {"bound": "hbm", "achieved": round(per_gpu, 1), "peak": pk["hbm"], "unit": "GB/s",
                             "frac": round(per_gpu / pk["hbm"], 4), "traffic": None,
                             "note": "per-GPU bytes read + written; with N > 1, (N-1)/N of the writes cross NVLink"},
                "cpu_baseline": None, "e2e": None, "gpu_launches": launches, "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_nw_band(args):
    """One NW alignment split by column bands over N GPUs (shard.NwBanded):
    each rank runs the wavefront over its strips, the band's left edge polled
    in the previous rank's memory over NVLink inside the kernel -- strong
    scaling; the check compares this rank's band with the single-GPU kernel.
    n = 65536 by default (LEGO_NW_BAND_N): at cfg4b's 16384 one GPU already
    holds all 128 strips at once, so bands cannot shorten the wavefront's
    critical path; at 65536 one GPU runs 512 strips in ~3.5 waves of 148."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2505_08091_b200 import kernels as K, shard
    world, rank, _local = dist_setup(args)
    if world == 1:                      # symmetric memory needs a process group, even of one rank
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0,
                                device_id=torch.device("cuda", 0))
    n = int(os.environ.get("LEGO_NW_BAND_N", "65536"))
    g = torch.Generator(device="cuda").manual_seed(4)
    sim = torch.randint(-10, 11, (n, n), generator=g, device="cuda", dtype=torch.int32)
    nb = shard.NwBanded(n, 1, sim.device)
    score = torch.empty(n + 1, n + 1, dtype=torch.int32, device="cuda")
    step = lambda: nb(sim, 10, out=score)  # noqa: E731
    step()
    torch.cuda.synchronize()
    whole = K.nw_score(sim, 10)
    lo, hi = 1 + 128 * nb.begin, min(n, 128 * nb.end) + 1
    ok = torch.equal(score[:, lo:hi], whole[:, lo:hi]) and torch.equal(score[0], whole[0])
    del whole
    launches0 = K.LAUNCHES[0]
    with ClockSampler(torch.cuda.current_device()) as clocks:
        ms = time_steps(step, args.steps, args.warmup, world)
    launches = K.LAUNCHES[0] - launches0 - 2 * args.warmup
    ms_step = ms / args.steps
    cells = n * n
    if rank == 0:
        line = {"metric": METRIC, "value": round(cells / (ms_step * 1e-3) / 1e9, 1), "unit": "GCUPS",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
                "data": "synthetic (uniform sim in [-10, 10], penalty 10)",
                "config": {"workload": f"cfg4b kernel on one {n}x{n} NW alignment in column bands over N GPUs "
                                       "(shard.NwBanded: the band's left edge polled in the peer's memory "
                                       "over NVLink inside the wavefront kernel)", "n": n,
                           "bands": nb.bands, "check_own_band": "ok" if ok else "MISMATCH",
                           "parallelism": f"strong: {world} column bands, edge hand-off inside the kernel"},
                "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": launches,
                "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def lower_size(layout):
    from paper_2505_08091_b200 import lower
    return lower.physical_size(layout)


def other_kernels(args, pk, world):
    """The remaining BASELINE configs, timed the same way (W warm-up, K steps)."""
    import torch

    import paper_2505_08091_b200 as L
    from paper_2505_08091_b200 import kernels as K
    res = {}
    steps, warm = max(5, min(args.steps, 50)), max(3, min(args.warmup, 5))

    def hbm_entry(name, nbytes, fn, traffic_key, extra=None):
        ms = time_steps(fn, steps, warm, world) / steps
        gbs = nbytes / (ms * 1e-3) / 1e9
        res[name] = {"GB/s": round(gbs, 1), "frac": round(gbs / pk["hbm"], 4),
                     "us": round(ms * 1e3, 1), "traffic": traffic_table().get(traffic_key),
                     **(extra or {})}

    # cfg1: 4096^2 fp32 tiled remap, batch 8 (512 MiB in, > L2)
    g1 = L.parse_layout("GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))")
    x1 = torch.randn(8, 4096 * 4096, device="cuda")
    y1 = torch.empty_like(x1)
    hbm_entry("cfg1_tiled_remap_fp32_b8", 2 * x1.numel() * 4,
              lambda: K.remap(x1, None, g1, out=y1), "remap_gather_fp32")
    del x1, y1
    # cfg3: softmax 8192^2 fp32 (256 MiB in: 2x L2)
    x3 = torch.randn(8192, 8192, device="cuda") * 4
    y3 = torch.empty_like(x3)
    hbm_entry("cfg3_softmax_fp32", 2 * x3.numel() * 4, lambda: K.softmax(x3, out=y3),
              "softmax_fp32")
    del x3, y3
    # cfg4a: antidiag remap 16384^2 int32
    g4 = L.parse_layout("GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))")
    x4 = torch.arange(16384 * 16384, device="cuda", dtype=torch.int32)
    y4 = torch.empty_like(x4)
    hbm_entry("cfg4a_antidiag_remap_i32", 2 * x4.numel() * 4,
              lambda: K.remap(x4, None, g4, out=y4), "remap_antidiag_i32",
              {"plan": repr(K.remap_plan(None, g4, 4))})
    del x4, y4
    # cfg4 index maps: every apply / inv of the antidiag layout (inv needs an exact isqrt)
    m4 = torch.empty(16384 * 16384, device="cuda", dtype=torch.int32)
    for which, fn in (("apply", K.apply_map), ("inv", K.inv_map)):
        ms = time_steps(lambda: fn(g4, out=m4), steps, warm, world) / steps
        res[f"cfg4_antidiag_{which}_map_i32"] = {
            "Gidx/s": round(m4.numel() / (ms * 1e-3) / 1e9, 1), "GB/s": round(m4.numel() * 4 / (ms * 1e-3) / 1e9, 1),
            "frac": round(m4.numel() * 4 / (ms * 1e-3) / 1e9 / pk["hbm"], 4), "us": round(ms * 1e3, 1)}
    del m4
    # SURVEY section 8(f) rows at scale (parity-tested in tests/): f1 multi-stage chain with an
    # in-tile GenP (Eq. (2) shape), f2 ExpandBy partial tiles, f4 injective scatter
    def frow(name, layout, n_elems, direction, dtype=torch.int32, scatter=False, traffic_key=None):
        x = torch.arange(n_elems, device="cuda", dtype=torch.int64).to(dtype)
        src_l, dst_l = (None, layout) if direction == "to" else (layout, None)
        out = K.remap(x, src_l, dst_l)
        # scatters into injective layouts run in fill mode: every destination
        # position written once (hits from the source, the rest the fill value)
        fill = 0 if scatter else None
        fn = lambda: K.remap(x, src_l, dst_l, out=out, fill=fill)  # noqa: E731
        plan = K.plan_remap(src_l, dst_l, x.element_size(), fill=scatter)
        # bytes: each source element read once, each destination element written once
        nbytes = (x.numel() + out.numel()) * x.element_size()
        hbm_entry(name, nbytes, fn, traffic_key, {"plan": repr(plan)})
        del x, out
    f1 = L.parse_layout("GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4]))"
                        ".OrderBy(RegP([128,128],[2,1]), GenP([64,64], antidiag))")
    frow("f1_chain_tile_antidiag_8192_i32", f1, 8192 * 8192, "to", traffic_key="remap_staged_f1_i32")
    f2 = L.parse_layout("ExpandBy([8000,8000],[8192,8192],"
                        "GroupBy([8192,8192]).OrderBy(RegP([128,64,128,64],[1,3,2,4])))")
    frow("f2_expand_partial_tiles_i32", f2, lower_size(f2), "from", traffic_key="remap_expand_f2_i32")
    even = L.GenP((1 << 26,), L.PermFn(lambda idx: idx[0] * 2, lambda idx: idx[0] * 2), None, name="even")
    f4 = L.GroupBy([1 << 26], orders=(L.OrderBy(even),), injective=True)
    frow("f4_injective_even_scatter_i32", f4, 1 << 26, "to", scatter=True,
         traffic_key="remap_scatter_f4_i32")
    # cfg4b: NW wavefront 16384^2 int32, driven by a LEGO layout of the cell grid
    try:
        from paper_2505_08091_b200 import nw as NW
        sim = torch.randint(-10, 11, (16384, 16384), device="cuda", dtype=torch.int32)
        score = torch.empty(16385, 16385, device="cuda", dtype=torch.int32)
        cells = 16384 * 16384
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from nw_perms import skew_order        # a user-defined GenP (rectangular anti-diagonal order)
        nw_layouts = [("cfg4b_nw_wavefront_i32", NW.nw_layout(16384)),
                      ("cfg4b_nw_tiles4096_user_skew_i32",
                       NW.nw_layout(16384, tile_rows=4096, tile_order=skew_order(4, 128))),
                      ("cfg4b_nw_tiles128_antidiag_i32", NW.nw_layout(16384, tile_rows=128, tile_order="antidiag"))]
        for name, lay in nw_layouts:
            K.nw_score(sim, 10, layout=lay, out=score)
            prog = NW.nw_program(lay, 16384)
            ms = time_steps(lambda: K.nw_score(sim, 10, layout=lay, out=score), 5, 3, world) / 5
            res[name] = {"GCUPS": round(cells / (ms * 1e-3) / 1e9, 1), "us": round(ms * 1e3, 1),
                         "GB/s": round((cells * 4 + 16385 ** 2 * 4) / (ms * 1e-3) / 1e9, 1),
                         "layout": NW.describe(lay),
                         "path": ("lego_nw_run (NVRTC program of the layout: " + str(prog.defines) + ")"
                                  if NW.needs_program(prog.defines) else
                                  "lego_nw_i32 (the layout lowers to no generated map: the library's "
                                  "built-in instance of the template)")}
        del sim, score
    except Exception as exc:  # noqa: BLE001
        res["cfg4b_nw_wavefront_i32"] = {"unavailable": str(exc)[:200]}
    # cfg5: bf16 GEMM 8192^3 on tcgen05
    try:
        a = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
        b = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
        c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
        ms = time_steps(lambda: K.gemm(a, b, out=c), steps, warm, world) / steps
        tf = 2 * 8192 ** 3 / (ms * 1e-3) / 1e12
        res["cfg5_gemm_bf16_8192"] = {"TFLOP/s": round(tf, 1), "frac": round(tf / pk["bf16"], 4),
                                      "frac_sustained": round(tf / pk["bf16_sustained"], 4),
                                      "us": round(ms * 1e3, 1)}
    except Exception as exc:  # noqa: BLE001
        res["cfg5_gemm_bf16_8192"] = {"unavailable": str(exc)[:200]}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="lego", choices=["lego", "reference"])
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="remap", choices=["remap", "gemm_b8", "transpose_shard", "nw_band"],
                    help="remap: headline cfg2 (weak scaling, one matrix per GPU); gemm_b8: cfg5 batch of 8 "
                         "8192^3 GEMMs split 8/N per GPU (strong); transpose_shard: one 16384^2 bf16 matrix "
                         "row-sharded over N GPUs into the Col layout by the fused routed transpose (strong); "
                         "nw_band: one 16384^2 NW alignment in column bands over N GPUs (strong)")
    ap.add_argument("--dry-run", action="store_true", help="launch and rendezvous only (CPU, gloo)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.workload == "gemm_b8":
        run_gemm_b8(args)
    elif args.workload == "transpose_shard":
        run_transpose_shard(args)
    elif args.workload == "nw_band":
        run_nw_band(args)
    else:
        run(args)


if __name__ == "__main__":
    main()
