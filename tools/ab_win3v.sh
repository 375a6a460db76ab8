# same-box A/B/C of exp/lib_{A,B,C}.so on the KLT launch for given windows (c5 data)
for i in 1 2; do for V in ${VS:-A B C}; do cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
  for w in ${@:-21}; do echo "$V $(python tools/klt_win_probe.py $w)"; done; done; done
