#!/bin/bash
# A/B sweep of SBGEMV layout knobs at C2 (run on the GPU box): NoTrans rows per
# thread, ConjTrans lanes per column, stage bytes.
for rpt in 1 2 4; do
  echo "RPT=$rpt"; FMV_SBGEMV_RPT=$rpt timeout 120 python tools/tune_sbgemv.py ${1:-ddddd} quick 2>&1 | grep "stages=3\|stages=6"
done
for lpc in 8 32; do
  echo "LPC=$lpc"; FMV_SBGEMV_LPC=$lpc timeout 120 python tools/tune_sbgemv.py ${1:-ddddd} quick 2>&1 | grep "stages=3\|stages=6"
done
