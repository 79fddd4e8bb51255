#!/bin/bash
# Fine sweep of the SBGEMV ring (stages x stage bytes) at C2 fp64, one CTA per SM.
for cfg in "4 32768" "5 24576" "4 28672" "3 40960" "4 36864" "5 28672" "3 45056" "4 40960" "3 49152" "2 65536"; do
  set -- $cfg
  FMV_SBGEMV_STAGES=$1 FMV_SBGEMV_STAGE_BYTES=$2 FMV_SBGEMV_CTAS_PER_SM=1 timeout 120 python tools/tune_sbgemv.py ddddd env 2>&1 | tail -1
done
