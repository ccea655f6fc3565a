# unfiltered initcheck over the sanitizer groups K (K2/K1/K3/K4) and S (streamer under train_epoch)
SEL_K="tests/test_stage_gpu.py tests/test_accum_gpu.py tests/test_optim_gpu.py"
SEL_S="tests/test_engine_gpu.py::test_host_streamed_equals_device_resident tests/test_engine_gpu.py::test_train_epoch_matches_reference tests/test_tracer_gpu.py"
for grp in K S; do
  eval sel=\$SEL_$grp
  timeout 1500 compute-sanitizer --tool initcheck --print-limit 20 --target-processes all --log-file gpurun_out/san_init3_${grp}.log \
      python -m pytest $sel -q -m gpu -p no:cacheprovider > gpurun_out/san_init3_${grp}.out 2>&1
  echo "initcheck $grp rc=$?" >> gpurun_out/san_init3_summary.txt
  tail -n 1 gpurun_out/san_init3_${grp}.out >> gpurun_out/san_init3_summary.txt
  grep -h "ERROR SUMMARY" gpurun_out/san_init3_${grp}.log >> gpurun_out/san_init3_summary.txt
  grep -h -A2 "Uninitialized" gpurun_out/san_init3_${grp}.log | grep " at " | sort | uniq -c | head -5 >> gpurun_out/san_init3_summary.txt
done
cat gpurun_out/san_init3_summary.txt
bash tools/runs/r02_k2_ab.sh
