#!/usr/bin/env bash
# Build variants of ONE translation unit and link each against the production
# objects (paper_2409_03686_b200/_build/*.o) into variants/lib_<tag>.so, for
# A/B runs on the GPU box with EXITMEASURE_B200_LIB=variants/lib_<tag>.so:
#   tools/diag/x2_variants.sh walk_f32x2 b3 "-DEM_X2_BLOCKS=3"  [more tag/flags pairs]
set -e
UNIT=$1; shift
B=paper_2409_03686_b200/_build
mkdir -p variants
MATH="-fmad=true -prec-sqrt=false -prec-div=false"; [ "$UNIT" = "capi" ] && MATH=""
KN="-DEM_BATCH_STEPS=8 -DEM_MIN_BLOCKS=0 -DEM_ANGLE_BITS=16 -DEM_Z_BITS=16 -DEM_TAB_WARP=0 -DEM_ROLL2_BLOCKS=4 -DEM_ROLL2_DYN=0 -DEM_POST_STOP=1 -DEM_TANG_K=4 -DEM_ROLL2_ONE=1"
while [ $# -gt 0 ]; do
  TAG=$1; FL=$2; shift 2
  (
  nvcc -c paper_2409_03686_b200/csrc/$UNIT.cu -o variants/${UNIT}_$TAG.o -gencode arch=compute_100a,code=sm_100a \
    -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include $MATH $KN $FL
  OBJS=$(ls $B/*.o | grep -v "/$UNIT.o")
  nvcc -shared -o variants/lib_$TAG.so $OBJS variants/${UNIT}_$TAG.o -gencode arch=compute_100a,code=sm_100a -cudart static -lpthread
  echo "built variants/lib_$TAG.so"
  ) &
done
wait
