# Build an alternate libvslam2d.so into exp/lib_$1.so with extra nvcc flags (A/B runs).
# usage: bash tools/build_variant.sh A "-DFOO"
mkdir -p exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC \
  -Xptxas -O3 $2 -I include -I paper_2506_04359_b200/csrc -o exp/lib_$1.so \
  paper_2506_04359_b200/csrc/*.cu -lcudart
