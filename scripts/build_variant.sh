#!/bin/bash
# Build a diagnostic / tuning variant of libpsso.so into variants/ (not the product):
#   scripts/build_variant.sh NAME "-DFLAG=1 ..."     then   PSSO_LIB=variants/libpsso_NAME.so python ...
set -e
cd "$(dirname "$0")/../paper_2110_01470_b200/csrc"
name=$1; flags=$2
bdir=/tmp/psso_build_$name; mkdir -p $bdir /tmp/psso_variants
for f in psso_api.cu psso_tiles_f64_ref.cu psso_tiles_f64_philox.cu psso_tiles_f32_ref.cu psso_tiles_f32_philox.cu \
         psso_swarm_f64_ref.cu psso_swarm_f64_philox.cu psso_swarm_f32_ref.cu psso_swarm_f32_philox.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC -I../../include $flags -c $f -o $bdir/${f%.cu}.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/psso_variants/libpsso_$name.so $bdir/*.o
rm -rf $bdir
echo built /tmp/psso_variants/libpsso_$name.so
