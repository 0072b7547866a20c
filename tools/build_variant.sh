#!/bin/bash
# Experiment build of the library with extra defines, e.g.
#   bash tools/build_variant.sh noticket -DSTC_EXPERIMENT_NOTICKET
# -> build_exp/libstc_noticket.so  (load with STC_LIBRARY=build_exp/libstc_noticket.so)
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build_exp/$name
mkdir -p "$out"
cd "$root/paper_1704_03092_b200/csrc"
for f in stc_kernels stc_gemm stc_fused stc_capi stc_host; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
    -c -o "$out/$f.o" $f.cu &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build_exp/lib$name.so" "$out"/*.o
echo "built build_exp/lib$name.so"
