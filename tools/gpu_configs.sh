# bench every config at N=1 plus the all-core oracle (GPU box).
mkdir -p gpurun_out
for CFG in c1 c2 c3 c4 c5; do
  timeout 900 python bench.py --config $CFG --steps 50 --warmup 5 > gpurun_out/cfg_$CFG.log 2>&1; echo $CFG=$?
done
for CFG in c2 c5; do
  timeout 300 python tools/oracle_allcores.py $CFG 15 > gpurun_out/allcores_$CFG.log 2>&1; echo all_$CFG=$?
done
nproc; lscpu | grep -E "Model name|^CPU\(s\)" 
