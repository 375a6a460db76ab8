# Round-2 profile capture at the bench default (c5): launch list + one ncu --set full
# capture per kernel.  usage: bash tools/gpu_profile_r02.sh [config] [tag]
CFG=${1:-c5}; TAG=${2:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --config $CFG --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$B > gpurun_out/${TAG}_plain_$CFG.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_$CFG.csv $B > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list=$?
for K in klt_kernel gftt_dense_kernel gftt_select pyramid_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -f -o gpurun_out/${TAG}_full_${CFG}_$K $B > gpurun_out/${TAG}_ncu_$K.log 2>&1; echo $K=$?
done
ls -la gpurun_out | grep $TAG
