# usage: bash tools/gpu_check.sh [ncu]   (run on the GPU box via gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c5.log 2>&1; echo bench=$?
timeout 900 python bench.py --config c2 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench2=$?
bash tools/gpu_multirank_smoke.sh
if [ "$1" = "ncu" ]; then
  B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
  $B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
fi
tail -2 gpurun_out/smoke.log | cut -c1-600
grep -E "passed|failed|KLT parity summary" gpurun_out/pytest_gpu.log | tail -3
grep -E "^FAILED|^E " gpurun_out/pytest_gpu.log | head -20 | cut -c1-500
python - <<'PY'
import json
for f in ("gpurun_out/bench_c5.log", "gpurun_out/bench_c2.log"):
    try:
        l = [x for x in open(f) if x.startswith("{")][-1]
        d = json.loads(l)
        print(f, "value", round(d["value"]), "ms/step", round(d["ms_per_step"], 3), "kpt/s", round(d["keypoints_tracked_per_s"]),
              {k: round(v["ms_per_launch"], 4) for k, v in d["kernels"].items()}, "roof", round(d["roofline"]["frac"], 4),
              "e2e", d.get("e2e") and round(d["e2e"]["value"]), "clk", d["clocks"], "cpu", d.get("cpu_baseline", {}).get("value"))
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-1500:])
PY
