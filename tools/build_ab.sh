# A/B builds for same-box comparisons: exp/lib_A.so from the working tree,
# exp/lib_B.so from the working tree with the listed files taken from git REV.
# usage: bash tools/build_ab.sh REV file1 [file2 ...]
REV=$1; shift
mkdir -p exp/b_src
rm -rf exp/b_src/*
cp -r paper_2506_04359_b200/csrc exp/b_src/csrc
for f in "$@"; do git show $REV:$f > exp/b_src/csrc/$(basename $f); done
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC -Xptxas -O3 -I include"
nvcc $F -I paper_2506_04359_b200/csrc -o exp/lib_A.so paper_2506_04359_b200/csrc/*.cu -lcudart &
nvcc $F -I exp/b_src/csrc -o exp/lib_B.so exp/b_src/csrc/*.cu -lcudart &
wait
ls -la exp/*.so
