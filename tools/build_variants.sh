#!/bin/bash
# Build K1 geometry variants of libpft_b200.so into variants/ (development A/B aid).
set -e
cd "$(dirname "$0")/.."
mkdir -p ${VARIANT_DIR:-variants}
[ -n "$SKIP_MAIN" ] || python -m paper_2008_12559_b200.build >/dev/null
FLAGS="-std=c++20 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-fopenmp -I include -I paper_2008_12559_b200/csrc -I paper_2008_12559_b200/build/gen"
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  D=""; for d in ${defs//,/ }; do D="$D -D$d"; done
  ( nvcc $FLAGS $D -c paper_2008_12559_b200/csrc/device/pft_kernels.cu -o /tmp/vk_$name.o &&
    nvcc $FLAGS $D -c paper_2008_12559_b200/csrc/device/pft_device.cu -o /tmp/vd_$name.o &&
    nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ${VARIANT_DIR:-variants}/lib_$name.so /tmp/vk_$name.o /tmp/vd_$name.o \
      paper_2008_12559_b200/build/host_*.o -Xcompiler -fopenmp -lgomp && echo "built $name" ) &
done
wait
