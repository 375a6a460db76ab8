# Same-box A/B of two library builds: alternates exp/lib_A.so and exp/lib_B.so
# (KLT probe, full iteration cap) so box-to-box clock differences cancel.
# usage: bash tools/ab_probe.sh [config ...]   (default c2)
CFGS=${@:-c2}
for CFG in $CFGS; do
  for i in 1 2; do
    for V in A B; do
      cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so
      echo "$CFG $V $(python tools/klt_probe.py $CFG 2>&1 | sed -n 5p)"
    done
  done
done
