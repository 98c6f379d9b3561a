#!/bin/bash
# Build a tuning variant of libvitdec_b200.so into build_variants/<name>/ with
# extra nvcc flags (A/B kernel runs: VITDEC_LIB=build_variants/<name>/libvitdec_b200.so).
#   tools/build_variant.sh myvariant -DSOME_MACRO=1   (run make first: vd_jit.cu includes build/vd_jit_sources.inc)
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
out=$ROOT/build_variants/$name
mkdir -p "$out"
SRC=$ROOT/paper_2011_09337_b200/csrc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$ROOT/include -I$ROOT/third_party/eigen_shim -I$SRC -I$ROOT/paper_2011_09337_b200/build $*"
pids=()
for src0 in $SRC/*.cu; do
  f=$(basename $src0 .cu)
  src=$src0; [ "$f" = vd_fast ] && [ -n "$FAST_SRC" ] && src=$FAST_SRC
  nvcc $FL -c $src -o $out/$f.o & pids+=($!)
done
g++ -O2 -fPIC -std=c++17 -I$ROOT/include -I$ROOT/third_party/eigen_shim -I$SRC -I/usr/local/cuda/include -c $SRC/vitdec_api.cpp -o $out/vitdec_api.o
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $out/libvitdec_b200.so $out/*.o -lpthread -ldl
echo built $out/libvitdec_b200.so
