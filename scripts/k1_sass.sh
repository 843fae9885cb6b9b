#!/bin/bash
# Dump the NVRTC K1 source of a config's model and its sm_100a SASS (no GPU needed).
# usage: SSA_K1_GEN=... SEED=<seed|-1> bash scripts/k1_sass.sh <config> <block> <minb> <outdir>
CFG=${1:-2}; BLK=${2:-128}; MINB=${3:-4}; OUT=${4:-/tmp/sass}
mkdir -p $OUT
python - <<PY
import inputs
from paper_1007_1768_b200 import ssa as S
m = S.Model(inputs.config($CFG).network)
open('$OUT/k1.cu', 'w').write(m.k1_source($BLK, $MINB, seed=int('${SEED:--1}')))
PY
nvcc -cubin -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -DSSA_NVRTC=1 -Xptxas -v \
  $OUT/k1.cu -o $OUT/k1.cubin 2>&1 | grep -E "registers|error" | head -3
cuobjdump -sass $OUT/k1.cubin | sed -n '/Function : ssa_k1/,$p' | grep -E "^\s+/\*[0-9a-f]{4}\*/" \
  | sed -E 's@ +/\* 0x[0-9a-f]+ \*/@@; s/ +;/;/; s/^ +//' > $OUT/k1.s
echo "instructions: $(wc -l < $OUT/k1.s)"
