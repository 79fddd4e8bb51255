#!/bin/bash
# fp16 ('h') NoTrans staging sweep at C2 (one CTA per SM build)
for cfg in "4 32768" "3 49152" "4 49152" "3 65536" "6 32768" "8 24576" "3 98304"; do
  set -- $cfg
  echo "stages=$1 bytes=$2"; FMV_SBGEMV_STAGES=$1 FMV_SBGEMV_STAGE_BYTES=$2 FMV_SBGEMV_CTAS_PER_SM=1 timeout 120 python tools/tune_sbgemv.py ddhdd,dssdd env 2>&1 | tail -2
done
