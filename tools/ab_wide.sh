#!/bin/bash
# SBGEMV: 2 CTAs/SM x 256 consumers (default build) vs 1 CTA/SM x 512 consumers
# (build/alt/lib_c512.so, -DFMV_SBGEMV_CONS=512 -DFMV_SBGEMV_MINB=1) at C2.
run() { FMV_SBGEMV_STAGES=$1 FMV_SBGEMV_STAGE_BYTES=$2 FMV_SBGEMV_CTAS_PER_SM=$3 timeout 120 python tools/tune_sbgemv.py ${CFG:-ddddd} env 2>&1 | tail -1; }
echo "default"; run 3 32768 2
for cfg in "3 32768" "4 32768" "3 49152" "6 32768" "4 49152" "3 65536"; do
  echo "c512 $cfg"; FMV_LIB_PATH=build/alt/lib_c512.so run $cfg 1
done
echo "default"; run 3 32768 2
