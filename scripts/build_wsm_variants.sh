#!/bin/bash
# Forecaster knob sweep: rebuild predictor.cu with -D overrides and link a variant library per
# setting (paper_2502_04077_b200/lib/variants/<name>.so; select with ATTNPRED_LIB=...).
#   scripts/build_wsm_variants.sh name:DEF=1,DEF2=3 ...
#   SRC=topk scripts/build_wsm_variants.sh ...   (rebuild csrc/topk.cu instead of predictor.cu)
set -e
cd "$(dirname "$0")/.."
LIB=paper_2502_04077_b200/lib
mkdir -p $LIB/variants
FL="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
SRC=${SRC:-predictor}
others=$(ls $LIB/obj/*.o | grep -v "/$SRC.o")
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  D=""; IFS=',' read -ra kv <<< "$defs"; for d in "${kv[@]}"; do D="$D -D$d"; done
  ( nvcc $FL $D -c paper_2502_04077_b200/csrc/$SRC.cu -o /tmp/${SRC}_$name.o && \
    nvcc -shared -cudart static -gencode arch=compute_100a,code=sm_100a $others /tmp/${SRC}_$name.o \
      -o $LIB/variants/$name.so && echo built $name ) &
done
wait
