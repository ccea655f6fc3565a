#!/bin/bash
# K5 cooperative-path size limit A/B in graph mode (bench C2 value), interleaved x2
for rep in 1 2; do for mb in 0 16 64; do
  MBS_K5_FUSED_MB=$mb timeout 600 python bench.py --no-cpu-baseline --steps 6 > /tmp/kf_$mb.json 2> /tmp/kf_$mb.err
  python -c "
import json; d=json.load(open('/tmp/kf_$mb.json')); print('MB=$mb', round(d['value']), round(d['e2e']['value']))"
  grep -i "capture failed" /tmp/kf_$mb.err | head -1
done; done
