"""Time the REFERENCE's own per-element Python path here.

The reference package is pure Python and exists only in this build
container (/root/reference is absent on the GPU box), so its CPU rate is
measured here, the way BASELINE.md asks: ``layout.apply`` per element over a
2^20-point sample of each bench layout, on multiprocessing.Pool(all cores);
the result (with the host's CPU model and core count) goes to
profiles/r02_reference_python.json.  bench.py's reference arm times the C
port (oracle/lego_oracle.c) on the GPU box's host, which is faster -- so the
GPU/CPU ratios it reports are conservative.
"""
import json
import multiprocessing as mp
import os
import platform
import subprocess
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import lego  # noqa: E402  (the reference)

LAYOUTS = {
    "cfg1": "GroupBy([4096,4096]).OrderBy(RegP([128,32,128,32],[1,3,2,4]))",
    "cfg2": "GroupBy([16384,16384]).OrderBy(Col(16384,16384))",
    "cfg4": "GroupBy([16384,16384]).OrderBy(GenP([16384,16384], antidiag))",
}
SAMPLE = 1 << 20
_L = None


def _chunk(bounds):
    lo, hi = bounds
    dims = _L.dims
    acc = 0
    for x in range(lo, hi):
        acc ^= _L.apply(lego.canon_unflatten(dims, x))
    return acc


def main():
    global _L
    cores = len(os.sched_getaffinity(0))
    out = {"cpu": platform.processor() or "", "cores": cores, "sample_points": SAMPLE, "layouts": {}}
    try:
        out["lscpu_model"] = [ln.split(":", 1)[1].strip() for ln in subprocess.check_output(["lscpu"], text=True)
                              .splitlines() if ln.startswith("Model name")][0]
    except Exception:  # noqa: BLE001
        pass
    for name, dsl in LAYOUTS.items():
        _L = lego.parse_layout(dsl)
        step = SAMPLE // (cores * 8)
        chunks = [(lo, lo + step) for lo in range(0, SAMPLE, step)]
        with mp.get_context("fork").Pool(cores) as pool:
            t0 = time.perf_counter()
            pool.map(_chunk, chunks)
            dt = time.perf_counter() - t0
        rate = SAMPLE / dt
        out["layouts"][name] = {"dsl": dsl, "elements_per_s": round(rate), "seconds": round(dt, 3),
                                "us_per_element_per_core": round(dt * cores / SAMPLE * 1e6, 3)}
        print(name, out["layouts"][name], flush=True)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "r02_reference_python.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
