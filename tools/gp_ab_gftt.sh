# Same-box A/B of K2 (exp/lib_A.so vs exp/lib_B.so): event time of v2d_detect_gftt and the
# ncu per-pass split (pass A / pass B, serialised replay) at c5 and c2.
for V in ${VS:-A B}; do cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
 for C in ${CFGS:-c5 c2}; do python tools/gftt_probe.py $C 20 | sed "s/^/$V /"
  ncu -k regex:gftt --metrics gpu__time_duration.sum --clock-control none -c 4 --csv python tools/gftt_probe.py $C 2 2>/dev/null | grep gpu__time | python -c "
import csv, sys
for r in csv.reader(sys.stdin):
    print('$V $C', r[4].split('(')[0].split('::')[-1], r[-1])"
 done; done
