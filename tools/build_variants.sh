#!/usr/bin/env bash
# Build libshplb variants of kernel 3 with different -D flags (dev tool).
# usage: [K3=persist] tools/build_variants.sh NAME "FLAGS" [NAME "FLAGS" ...]
# -> paper_2603_10353_b200/lib/variants/libshplb_NAME.so (needs a prior `make` in csrc/);
# K3=persist rebuilds the persistent CTA-pair kernel (fa_persist_sm100.cu) with FLAGS
# instead of fa_sm100.cu.
set -euo pipefail
cd "$(dirname "$0")/../paper_2603_10353_b200/csrc"
OUT=../lib/variants
mkdir -p "$OUT"
pids=()
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  case "${K3:-single}" in
    persist) src=kernels/fa_persist_sm100.cu; keep="../lib/obj/kernels/fa_sm100.o";;
    *) src=kernels/fa_sm100.cu; keep="../lib/obj/kernels/fa_persist_sm100.o";;
  esac
  (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
      -I../../include -I/usr/local/cuda/include --expt-relaxed-constexpr $flags -c $src -o "$OUT/fa_$name.o" &&
   g++ -shared -o "$OUT/libshplb_$name.so" ../lib/obj/kernels/estimator.o ../lib/obj/kernels/profiler.o "$OUT/fa_$name.o" $keep \
      ../lib/obj/shplb_api.o ../lib/obj/host/*.o -L/usr/local/cuda/lib64 -lcudart_static -lrt \
      -ldl -lpthread -fopenmp && echo "built $name") &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
