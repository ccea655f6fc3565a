# compute-sanitizer over the model-side kernels of the benched stack: K5 BatchNorm (TMA ring, cooperative
# launches, PDL), K6 max-pool / skip join, K7 stem im2col
SEL="tests/test_bn_gpu.py tests/test_pool_gpu.py tests/test_stem_gpu.py"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-name kns=3mbs --target-processes all --print-limit 50 \
      --log-file gpurun_out/san_mo_${tool}_%p.log python -m pytest $SEL -q -m gpu -p no:cacheprovider -x \
      > gpurun_out/san_mo_${tool}.out 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_mo_summary.txt
  tail -n 2 gpurun_out/san_mo_${tool}.out >> gpurun_out/san_mo_summary.txt
  grep -h "SUMMARY" gpurun_out/san_mo_${tool}_*.log | sort | uniq -c >> gpurun_out/san_mo_summary.txt
done
cat gpurun_out/san_mo_summary.txt
