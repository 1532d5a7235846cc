#!/bin/bash
# Build tuning variants of libpsso.so into variants/ (PSSO_LIB=... selects one at run time).
#   scripts/build_variants.sh name1:"-DFOO=1 -DBAR=2" name2:"..."
set -e
cd "$(dirname "$0")/../paper_2110_01470_b200/csrc"
mkdir -p ../../variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  out=../../variants/libpsso_$name.so
  bdir=build_$name; mkdir -p $bdir
  for f in psso_api.cu psso_tiles_f64_ref.cu psso_tiles_f64_philox.cu psso_tiles_f32_ref.cu psso_tiles_f32_philox.cu; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
      -Xcompiler -fPIC -I../../include $flags -c $f -o $bdir/${f%.cu}.o &
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $bdir/*.o
  rm -rf $bdir
  echo built $out
done
