# Same-box A/B of the K2 || K3 stream overlap (bench --overlap 1 vs 0).
for CFG in ${@:-c5 c2}; do
  for i in 1 2; do
    for O in 1 0; do
      python bench.py --config $CFG --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --overlap $O 2>&1 | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', 'overlap=$O', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_launch'], 4) for k, v in d['kernels'].items()})"
    done
  done
done
