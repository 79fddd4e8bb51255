#!/bin/bash
# Block SBGEMV: 2 x 256-consumer CTAs per SM vs 1 x 512 (build/alt/lib_blk{256,512}.so), stage sizes.
for v in 256 512; do
  for sb in 32768 49152 65536; do
    echo "blk$v stage $sb"; FMV_LIB_PATH=build/alt/lib_blk$v.so FMV_BLOCK_STAGE_BYTES=$sb timeout 200 python tools/bench_block.py ddddd 4,8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  K=%d F %.0f RHS/s (%.0f GB/s)  F* %.0f RHS/s (%.0f GB/s)' % (d['K'], d['F']['rhs_per_s'], d['F']['op_stream_gbs'], d['Fstar']['rhs_per_s'], d['Fstar']['op_stream_gbs']))"
  done
done
