# K1 bf16-assign unroll A/B + K2 CTAs/SM A/B (kbench, events) and ncu; K1C per-rank sanitizer; bench-stack
# parity report; the full GPU suite
for v in default u4 tile16k; do
  case $v in
    default) env="MBS_AB=0";;
    u4) env="MBS_NATIVE_LIB=$PWD/ab/libmbs_k1u4.so";;
    tile16k) env="MBS_K1_TILE=16384";;
  esac
  env $env timeout 300 python tools/kbench.py --config c2 > gpurun_out/c4_kbench_$v.json 2>&1
done
for c in 2 3 4; do MBS_K2_CTAS_PER_SM=$c timeout 300 python tools/kbench.py --config c2 > gpurun_out/c4_kbench_k2cta$c.json 2>&1; done
python - <<'PY'
import json
for v in ["default","u4","tile16k","k2cta2","k2cta3","k2cta4"]:
    try:
        d=json.load(open(f"gpurun_out/c4_kbench_{v}.json"))
        print(v, {k: round(x["us_median"],2) for k,x in d.items() if isinstance(x,dict) and k.startswith(("k1","k2_stage_u8_bf16"))})
    except Exception as e: print(v, "ERR", e)
PY
for c in 2 3; do
  MBS_K2_CTAS_PER_SM=$c timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stage|k_accum" -c 8 --csv \
      --log-file gpurun_out/c4_k2cta${c}.csv python tools/profile_step.py > /dev/null 2>&1
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stage|k_accum" -c 8 --csv \
    --log-file gpurun_out/c4_default.csv python tools/profile_step.py > /dev/null 2>&1
MBS_NATIVE_LIB=$PWD/ab/libmbs_k1u4.so timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stage|k_accum" -c 8 --csv \
    --log-file gpurun_out/c4_u4.csv python tools/profile_step.py > /dev/null 2>&1
bash tools/runs/r02_sanitize_k1c.sh
MBS_PARITY_REPORT=$PWD/gpurun_out/parity_report.jsonl timeout 1200 python -m pytest tests/test_bench_stack_parity_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/c4_parity.log 2>&1; tail -3 gpurun_out/c4_parity.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/c4_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/c4_pytest_gpu.log; tail -4 gpurun_out/c4_pytest_gpu.log
