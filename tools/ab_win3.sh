# same-box comparison of several builds on the KLT launch (c5 data): bash tools/ab_win3.sh "A R112 R120" 21
VS=$1; shift
for i in 1 2; do for V in $VS; do cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
  for w in ${@:-21}; do echo "$V $(python tools/klt_win_probe.py $w)"; done; done; done
