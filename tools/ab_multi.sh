# Same-box comparison of several builds exp/lib_<V>.so x bench options.
# usage: bash tools/ab_multi.sh "A P2 P3" "--overlap 0|--overlap 1" c5 c2
VS=$1; OPTS=$2; shift 2
IFS="|" read -ra OA <<< "$OPTS"; [ ${#OA[@]} -eq 0 ] && OA=("")
for CFG in ${@:-c5}; do
  for i in 1 2; do
    for V in $VS; do
      for O in "${OA[@]}"; do
        cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
        python bench.py --config $CFG --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $O 2>&1 | tail -1 | \
          python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', '$V', '$O', round(d['value']), round(d['ms_per_step'],4), {k: round(v['ms_per_launch'], 4) for k, v in d['kernels'].items()})"
      done
    done
  done
done
