#!/bin/bash
# Build the library from a git revision (default HEAD) as lib/variants/libetap_mla_<name>.so for
# same-box A/B runs: bash scripts/build_head_variant.sh <name> [rev]
NAME=$1; REV=${2:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p $TMP/include $TMP/pkg/csrc
for f in etap_mla.cu etap_peer.cu etap_proj.cu etap_fp8.cu etap_mla_host.cpp sm100_ptx.cuh etap_mla_kernels.cuh etap_fp8.cuh; do
  git -C $ROOT show $REV:paper_2506_01969_b200/csrc/$f > $TMP/pkg/csrc/$f
done
git -C $ROOT show $REV:include/etap_mla.h > $TMP/include/etap_mla.h
mkdir -p $ROOT/paper_2506_01969_b200/lib/variants
cd $TMP/pkg/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -shared etap_mla.cu etap_peer.cu etap_proj.cu etap_fp8.cu etap_mla_host.cpp \
  -o $ROOT/paper_2506_01969_b200/lib/variants/libetap_mla_$NAME.so -Xlinker --export-dynamic \
  -Xlinker --version-script=$ROOT/paper_2506_01969_b200/lib/exports.map
rm -rf $TMP
