set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; tail -3 gpurun_out/pytest_gpu_final.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; cat gpurun_out/smoke_final.log
timeout 600 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
timeout 1500 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r01_c2_v9_launches.csv python tools/profile_step.py > /dev/null 2>&1
python -c "
import json
for f in ['gpurun_out/final_c2.json','gpurun_out/final_c4.json']:
    d=json.load(open(f)); print(f, d['value'], d.get('e2e',{}).get('value'), (d.get('no_stream') or {}).get('value'), (d.get('no_stream_torch_ops') or {}).get('value'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))
"
