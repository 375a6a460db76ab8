# Final round-2 evidence on one GPU box (run via gpurun): build, smoke, GPU suite, the
# default bench line (what the driver runs), c1-c4 lines, c5 variants, the reference arm,
# multi-rank (gloo, one GPU) c5 and c2, and the c5 launch list + ncu full per kernel.
# usage: bash tools/gpu_final_r02.sh [tag=r02h]
TAG=${1:-r02h}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.log 2>&1; echo bench_default=$?
for CFG in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $CFG --steps 50 --warmup 5 > gpurun_out/${TAG}_bench_$CFG.log 2>&1; echo $CFG=$?
done
timeout 900 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --extras > gpurun_out/${TAG}_extras.log 2>&1; echo extras=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.log 2>&1; echo ref=$?
bash tools/gpu_multirank_smoke.sh c5 > /dev/null 2>&1; cp gpurun_out/multirank_c5.log gpurun_out/${TAG}_multirank_c5.log
bash tools/gpu_multirank_smoke.sh c2 > /dev/null 2>&1; cp gpurun_out/multirank_c2.log gpurun_out/${TAG}_multirank_c2.log
bash tools/gpu_profile_r02.sh c5 $TAG > /dev/null 2>&1; echo profile=$?
tail -2 gpurun_out/${TAG}_smoke.log | cut -c1-300; grep -E "passed|failed|KLT parity summary" gpurun_out/${TAG}_pytest_gpu.log | tail -2
