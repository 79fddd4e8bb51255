#!/bin/bash
# SBGEMV residency A/B at C2: the default build (2 CTAs/SM) vs a build sized for
# 3 CTAs/SM (-DFMV_SBGEMV_MINB=3, build/alt/lib_minb3.so) at several stage sizes.
q() { timeout 120 python tools/tune_sbgemv.py ddddd quick 2>&1 | grep "stages=3 bytes= 32768"; }
echo "default 2/SM"; q
for sb in 20480 24576 16384; do
  for st in 3 4; do
    echo "minb3 3/SM stage $sb x $st"
    FMV_LIB_PATH=build/alt/lib_minb3.so FMV_SBGEMV_CTAS_PER_SM=3 FMV_SBGEMV_STAGE_BYTES=$sb FMV_SBGEMV_STAGES=$st \
      timeout 120 python tools/tune_sbgemv.py ddddd quick 2>&1 | grep "stages=3 bytes= 32768"
  done
done
echo "default 2/SM"; q
