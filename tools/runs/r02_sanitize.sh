# compute-sanitizer over this repo's kernels (mangled names contain "3mbs": namespace mbs) on the K2 bulk ring,
# K1/K3/K4, the host streamer paths and the K1C two-process peer all-reduce. Summaries -> gpurun_out/san_*.
SEL_K="tests/test_stage_gpu.py tests/test_accum_gpu.py tests/test_optim_gpu.py"
SEL_S="tests/test_engine_gpu.py::test_host_streamed_equals_device_resident tests/test_engine_gpu.py::test_train_epoch_matches_reference tests/test_tracer_gpu.py"
SEL_P="tests/test_dp_gpu.py::test_fused_peer_allreduce_two_ranks_one_gpu"
for tool in memcheck racecheck synccheck initcheck; do
  for grp in K S P; do
    eval sel=\$SEL_$grp
    timeout 700 compute-sanitizer --tool $tool --kernel-name kns=3mbs --target-processes all --print-limit 50 \
        --log-file gpurun_out/san_${tool}_${grp}_%p.log \
        python -m pytest $sel -q -m gpu -p no:cacheprovider > gpurun_out/san_${tool}_${grp}.out 2>&1
    echo "$tool $grp rc=$?" >> gpurun_out/san_summary.txt
    tail -n 2 gpurun_out/san_${tool}_${grp}.out >> gpurun_out/san_summary.txt
    grep -h "ERROR SUMMARY" gpurun_out/san_${tool}_${grp}_*.log | sort | uniq -c >> gpurun_out/san_summary.txt
  done
done
cat gpurun_out/san_summary.txt
