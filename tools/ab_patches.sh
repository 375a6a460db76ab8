# same-box A/B of the f4 patches kernel: exp/lib_<V>.so for V in $VS (default A B)
for i in 1 2; do for V in ${VS:-A B}; do cp exp/lib_$V.so paper_2506_04359_b200/libvslam2d.so; echo "$V $(python tools/patches_probe.py)"; done; done
