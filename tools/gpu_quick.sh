# Quick GPU check after a kernel change: build, smoke, a pytest selection, short benches.
# usage: bash tools/gpu_quick.sh "<pytest -k expr or test files>"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/q_smoke.log | cut -c1-300
timeout 1500 python -m pytest $1 -q -p no:cacheprovider -x > gpurun_out/q_pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|KLT parity summary" gpurun_out/q_pytest.log | tail -3
grep -E "^FAILED|^E " gpurun_out/q_pytest.log | head -10 | cut -c1-400
for C in c5 c2; do
timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench_$C.log 2>&1; echo bench_$C=$?
python - $C <<'PY'
import json, sys
f = "gpurun_out/q_bench_%s.log" % sys.argv[1]
try:
    d = json.loads([x for x in open(f) if x.startswith("{")][-1])
    print(f, "value", round(d["value"]), "ms/step", round(d["ms_per_step"], 4),
          {k: round(v["ms_per_launch"], 4) for k, v in d["kernels"].items()}, "roof", round(d["roofline"]["frac"], 4),
          "e2e", d.get("e2e") and round(d["e2e"]["value"]), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(f, "ERR", e, open(f).read()[-1500:])
PY
done
