# compute-sanitizer on BOTH ranks of the K1C peer all-reduce (each rank its own sanitized process)
for tool in memcheck racecheck synccheck; do
  port=$((29600 + RANDOM % 300))
  for r in 0 1; do
    timeout 900 compute-sanitizer --tool $tool --kernel-name kns=3mbs --print-limit 50 \
        --log-file gpurun_out/san_k1c_${tool}_r${r}.log python tools/k1c_rank.py $r $port /tmp/k1c_$tool \
        > gpurun_out/san_k1c_${tool}_r${r}.out 2>&1 &
  done
  wait
  python tools/k1c_rank.py check /tmp/k1c_$tool >> gpurun_out/san_k1c_summary.txt 2>&1
  echo "$tool:" >> gpurun_out/san_k1c_summary.txt
  grep -h "SUMMARY" gpurun_out/san_k1c_${tool}_r*.log >> gpurun_out/san_k1c_summary.txt
done
cat gpurun_out/san_k1c_summary.txt
