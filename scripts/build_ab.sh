# build .so variants for A/B: scripts/build_ab.sh name "-DFLAG ..." [name "-D..."]...
set -e
while [ $# -ge 2 ]; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -shared \
    $2 -I include -o scripts/_ab/$1.so paper_2412_13211_b200/csrc/trajlab_b200.cu &
  shift 2
done
wait
