#!/bin/bash
# Build the variants first, e.g.: (cd paper_2110_12484_b200/csrc && nvcc ... -DMBS_K1_MIXED_MINBLOCKS=3 -DMBS_K1_U8=2 -DMBS_K1_BF16_X4=0 -shared *.cu *.cpp -o ../../tools/k1ab/k1_a.so)
# K1 bf16-gradient (shadow-weight) variants A/B in the C2 pipeline: bench.py's live K1 timing per variant .so
for v in a b c d; do
  MBS_NATIVE_LIB=tools/k1ab/k1_$v.so timeout 600 python bench.py --no-cpu-baseline --steps 4 > /tmp/k1_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/k1_$v.json'))
print('$v', round(d['value']), 'K1 us', round(d['roofline']['avg_launch_us'], 1), 'frac', round(d['roofline']['frac'], 3))"
done
