# compute-sanitizer over tools/sanitize_case.py, ONE tool per call (after a clean plain run).
# usage: bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck|initcheck
T=${1:-memcheck}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1; echo plain=$?; tail -1 gpurun_out/san_plain.log
timeout 1500 compute-sanitizer --tool $T --error-exitcode 9 --print-limit 50 python tools/sanitize_case.py > gpurun_out/san_$T.log 2>&1; echo $T=$?
tail -6 gpurun_out/san_$T.log
