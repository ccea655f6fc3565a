# is initcheck blind to bulk-async (TMA) stores? the same staging test on a plain-store path (1) and the bulk path (4)
for p in 1 4; do
  MBS_K2_PATH=$p timeout 900 compute-sanitizer --tool initcheck --print-limit 5 --log-file gpurun_out/san_init4_p$p.log \
      python -m pytest tests/test_stage_gpu.py -q -m gpu -p no:cacheprovider -k "test_stage_bit_exact" > gpurun_out/san_init4_p$p.out 2>&1
  echo "MBS_K2_PATH=$p rc=$? $(tail -n 1 gpurun_out/san_init4_p$p.out)"; grep -h "ERROR SUMMARY" gpurun_out/san_init4_p$p.log
done
