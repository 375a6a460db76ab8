# same-box A/B of the §8(f) kernels (klt_win11 = pair kernel, f2, f3, f4) over builds exp/lib_<V>.so
# usage: bash tools/ab_extras.sh "A Q14" [config]
for i in 1 2; do for V in $1; do
  cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
  python bench.py --config ${2:-c5} --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --extras 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); x=d['variants']; print('$V', round(d['kernels']['klt']['ms_per_launch'],4), {k: round(v['ms_per_launch'],4) for k, v in x.items() if isinstance(v, dict) and 'ms_per_launch' in v})"
done; done
