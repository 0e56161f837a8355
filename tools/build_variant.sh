#!/bin/bash
# Build a tuning variant of libsqngd.so with extra -D flags (A/B runs: SQNGD_LIB=tools/variants/libsqngd_<name>.so).
#   bash tools/build_variant.sh <name> [-DSQNGD_X=1 ...]       (CSRC=<dir> overrides the kernel sources)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python -c "from paper_2604_25728_b200 import build as B; B.build()" > /dev/null
NCCL=$(python -c "from paper_2604_25728_b200 import build as B; print(B._nccl_path())")
mkdir -p tools/variants
C=paper_2604_25728_b200/csrc
S=${CSRC:-$C}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --std=c++17 -Xcompiler -fPIC -I include \
  -DSQNGD_NCCL_PATH="\"$NCCL\"" "$@" -c -o /tmp/sqngd_$name.o $S/sqngd.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/variants/libsqngd_$name.so /tmp/sqngd_$name.o $C/net.cu.o $C/run.cu.o -ldl
echo tools/variants/libsqngd_$name.so
