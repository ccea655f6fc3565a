# initcheck WITHOUT a kernel filter (a filtered run cannot see memory initialised by torch's own kernels and
# reports it as uninitialised), over small selections
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 --log-file gpurun_out/san_init2_optim.log \
    python -m pytest tests/test_optim_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/san_init2_optim.out 2>&1
echo "optim rc=$?"; tail -1 gpurun_out/san_init2_optim.out; grep -h "ERROR SUMMARY" gpurun_out/san_init2_optim.log
grep -h -A2 "Uninitialized" gpurun_out/san_init2_optim.log | grep " at " | sort | uniq -c | head
timeout 1500 compute-sanitizer --tool initcheck --print-limit 20 --log-file gpurun_out/san_init2_accum.log \
    python -m pytest tests/test_accum_gpu.py -q -m gpu -p no:cacheprovider -k "oracle and 16 or unit_factor or bucketed or unaligned" > gpurun_out/san_init2_accum.out 2>&1
echo "accum rc=$?"; tail -1 gpurun_out/san_init2_accum.out; grep -h "ERROR SUMMARY" gpurun_out/san_init2_accum.log
grep -h -A2 "Uninitialized" gpurun_out/san_init2_accum.log | grep " at " | sort | uniq -c | head
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 --log-file gpurun_out/san_init2_stage.log \
    python -m pytest tests/test_stage_gpu.py -q -m gpu -p no:cacheprovider -k "streamer_partition" > gpurun_out/san_init2_stage.out 2>&1
echo "stage rc=$?"; tail -1 gpurun_out/san_init2_stage.out; grep -h "ERROR SUMMARY" gpurun_out/san_init2_stage.log
grep -h -A2 "Uninitialized" gpurun_out/san_init2_stage.log | grep " at " | sort | uniq -c | head
