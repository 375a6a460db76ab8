# Round profile set (on the GPU box): launch list of the default bench command
# and one full capture per kernel at c2 (and c5 for gftt).  Outputs in gpurun_out/.
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_launch.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launch=$?
for K in klt gftt pyramid; do
  C=1; [ "$K" = gftt ] && C=2   # gftt: dense pass A + select pass B
  $B > gpurun_out/plain_$K.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c $C -o gpurun_out/full_c2_$K $B > gpurun_out/ncu_$K.log 2>&1; echo $K=$?
done
B5="python bench.py --config c5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$B5 > gpurun_out/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"klt|gftt" -s 2 -c 2 -o gpurun_out/full_c5 $B5 > gpurun_out/ncu_c5.log 2>&1; echo c5=$?
