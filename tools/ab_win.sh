# KLT launch time per window size for two builds (exp/lib_A.so, exp/lib_NP.so) on c5 data
for V in ${@:-A NP}; do
  cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --extras 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['variants']
print('$V', 'klt21', round(d['kernels']['klt']['ms_per_launch'],4), 'win11', round(v['klt_win11']['ms_per_launch'],4), 'gn/kp', round(v['klt_win11']['gn_steps_per_kp'],2), 'tracked', round(v['klt_win11']['tracked_fraction'],4))"
done
