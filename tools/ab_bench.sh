# Same-box A/B of two library builds on the whole bench step (all kernels):
# alternates exp/lib_A.so and exp/lib_B.so.  usage: bash tools/ab_bench.sh [config ...]
CFGS=${@:-c2}
for CFG in $CFGS; do
  for i in 1 2; do
    for V in A B; do
      cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
      python bench.py --config $CFG --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', '$V', round(d['value']), {k: round(v['ms_per_launch'], 4) for k, v in d['kernels'].items()})"
    done
  done
done
