"""Measure the dense FP8 tensor-core peak of this B200 the way MEASURED_PEAKS.json measures bf16:
a library GEMM (cuBLASLt through torch._scaled_mm, 8192^3, 2 N^3 flop), best of 10 (burst) and
back to back for ~4 s (sustained), with nvidia-smi clocks sampled during the sustained run.
E5M2 x E5M2 is not a cuBLASLt FP8 combination; the kind::f8f6f4 tensor pipe runs every 8-bit
format at the same rate, so E4M3 x E4M3 (and E5M2 x E4M3) measure the E5M2 peak. bf16 is
re-measured in the same run for the ratio. Writes one JSON object (stdout and --out)."""
import argparse
import json
import statistics
import subprocess
import threading
import time

import torch


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def sustained(fn, seconds):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    e0.record()
    t0 = time.time()
    while time.time() - t0 < seconds:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def clocks(stop, rows):
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,"
                              "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        if out:
            rows.append(out)
        stop.wait(0.2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    N = a.n
    flop = 2.0 * N ** 3
    res = {"n": N, "how": "torch._scaled_mm (cuBLASLt) NxNxN, 2N^3 flop; best of 10 (burst), "
                          "back to back ~4 s (sustained)"}
    A16 = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    B16 = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    f = lambda: torch.matmul(A16, B16)   # noqa: E731
    for _ in range(3):
        f()
    res["bf16_tflops"] = flop / timed(f, 10) / 1e9
    one = torch.ones((), device="cuda")
    combos = {"e4m3xe4m3": (torch.float8_e4m3fn, torch.float8_e4m3fn),
              "e5m2xe4m3": (torch.float8_e5m2, torch.float8_e4m3fn),
              "e5m2xe5m2": (torch.float8_e5m2, torch.float8_e5m2)}
    for name, (ta, tb) in combos.items():
        A = (torch.randn(N, N, device="cuda") * 0.5).to(ta)
        B = (torch.randn(N, N, device="cuda") * 0.5).to(tb).t()   # column-major B
        g = lambda: torch._scaled_mm(A, B, scale_a=one, scale_b=one,   # noqa: E731
                                     out_dtype=torch.bfloat16)
        try:
            for _ in range(3):
                g()
            torch.cuda.synchronize()
        except Exception as e:   # unsupported combination in cuBLASLt
            res[f"fp8_{name}"] = f"unsupported: {str(e).splitlines()[0][:120]}"
            continue
        res[f"fp8_{name}_tflops"] = flop / timed(g, 10) / 1e9
        if name == "e4m3xe4m3":
            rows, stop = [], threading.Event()
            th = threading.Thread(target=clocks, args=(stop, rows), daemon=True)
            th.start()
            ms = sustained(g, 4.0)
            stop.set()
            th.join()
            res["fp8_e4m3xe4m3_tflops_sustained"] = flop / ms / 1e9
            sm = [float(r.split(",")[0]) for r in rows if r.split(",")[0].strip().isdigit()]
            res["clocks_sustained"] = {"sm_mhz_median": statistics.median(sm) if sm else None,
                                       "samples": len(rows),
                                       "power_cap_active": any("Active" in r for r in rows)}
    rows, stop = [], threading.Event()
    res["bf16_tflops_sustained"] = flop / sustained(f, 4.0) / 1e9
    fp8 = res.get("fp8_e4m3xe4m3_tflops")
    if fp8:
        res["fp8_over_bf16_burst"] = fp8 / res["bf16_tflops"]
    res["gpu"] = torch.cuda.get_device_name()
    print(json.dumps(res))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
