# compute-sanitizer initcheck (uninitialised device reads) on this repo's kernels only, over a bounded selection
for grp in accum stage optim; do
  case $grp in
    accum) sel="tests/test_accum_gpu.py";;
    stage) sel="tests/test_stage_gpu.py -k every_path or streamer_partition";;
    optim) sel="tests/test_optim_gpu.py";;
  esac
  timeout 1500 compute-sanitizer --tool initcheck --kernel-name kns=3mbs --print-limit 20 \
      --log-file gpurun_out/san_init_${grp}.log python -m pytest $sel -q -m gpu -p no:cacheprovider > gpurun_out/san_init_${grp}.out 2>&1
  echo "$grp rc=$?" >> gpurun_out/san_init_summary.txt
  tail -n 1 gpurun_out/san_init_${grp}.out >> gpurun_out/san_init_summary.txt
  grep -h "ERROR SUMMARY" gpurun_out/san_init_${grp}.log >> gpurun_out/san_init_summary.txt
  grep -h -m3 -A3 "Uninitialized" gpurun_out/san_init_${grp}.log | grep -i "kernel\|mbs" | head -5 >> gpurun_out/san_init_summary.txt
done
cat gpurun_out/san_init_summary.txt
