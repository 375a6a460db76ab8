# same-box A/B of exp/lib_A.so vs exp/lib_B.so on the KLT launch for given windows (c5 data)
for i in 1 2; do for V in A B; do cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
  for w in ${@:-11}; do echo "$V $(python tools/klt_win_probe.py $w)"; done; done; done
