# usage: bash tools/gpu_ncu2.sh <config> <kernel-regex> <count> <outname>
mkdir -p gpurun_out
CFG=${1:-c2}; K=${2:-klt}; N=${3:-1}; OUT=${4:-prof}
B="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_$OUT.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"$K" -s 2 -c $N -o gpurun_out/$OUT $B > gpurun_out/ncu_$OUT.log 2>&1; echo ncu=$?
