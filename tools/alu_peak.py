#!/usr/bin/env python
"""Measure the CUDA-core roofline denominators on the B200 and write
profiles/alu_peaks.json (read by bench.py's peaks()).

    python tools/alu_peak.py            # on the GPU box (gpurun)

Builds tools/alu_peak.cu for sm_100a, runs it while nvidia-smi samples the SM
clock and throttle reasons (bench.py's Clocks), and records, per kernel,
lane-instructions/s and flop/s (FFMA2 = 4 flop per lane-instruction, FFMA = 2)
or integer lane-ops/s (IADD3).  The FP32 peak the KLT roofline uses is the
best fp32 rate (FFMA2, the instruction K3's inner loops are made of); the
integer lane-op peak K2's model uses is the IADD3 rate.
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import Clocks  # noqa: E402


def main():
    src = os.path.join(ROOT, "tools", "alu_peak.cu")
    exe = "/tmp/alu_peak_bin"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe, src],
                   check=True)
    subprocess.run([exe, "2"], check=True, capture_output=True)  # warm the GPU clocks
    clk = Clocks(0)
    t0 = time.time()
    out = subprocess.run([exe, "40"], check=True, capture_output=True, text=True).stdout
    rec = clk.stop()
    rows = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    by = {r["kernel"]: r for r in rows}
    res = {
        "ffma2_tflops": by["ffma2"]["ops_per_s"] / 1e12,
        "ffma_tflops": by["ffma"]["ops_per_s"] / 1e12,
        "ffma_imm_tflops": by["ffma_imm"]["ops_per_s"] / 1e12,
        "iadd3_tops": by["iadd3"]["ops_per_s"] / 1e12,
        "mixed_ffma2_iadd3_t_lane_instr": by["mixed_ffma2_iadd3"]["lane_instr_per_s"] / 1e12,
        "kernels": rows,
        "clocks": rec or {"sm_mhz": float("nan")},
        "seconds": time.time() - t0,
        "how": "tools/alu_peak.cu: 8 independent chains/thread, 4096 unrolled iterations, "
               "148 x 8 CTAs x 256 threads, best of 5 x 40 launches (CUDA events); "
               "clocks sampled by nvidia-smi during the run",
    }
    with open(os.path.join(ROOT, "profiles", "alu_peaks.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}))


if __name__ == "__main__":
    main()
