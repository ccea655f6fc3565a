# compute-sanitizer memcheck / racecheck / synccheck over the warp-specialised K2 (MBS_K2_PATH=5, 8 and 16 px per
# lane; every shape of the every-path test: ragged tiles, tiles across rows, one-tile CTAs)
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=3mbs --print-limit 50 --log-file gpurun_out/san_k2ws_${tool}.log \
      python -m pytest tests/test_stage_gpu.py -q -m gpu -p no:cacheprovider -k "every_path and (5 or ws16)" > gpurun_out/san_k2ws_${tool}.out 2>&1
  echo "$tool rc=$? $(tail -n 1 gpurun_out/san_k2ws_${tool}.out) | $(grep -h 'ERROR SUMMARY' gpurun_out/san_k2ws_${tool}.log | sort | uniq -c | tr '\n' ' ')" >> gpurun_out/san_k2ws_summary.txt
done
cat gpurun_out/san_k2ws_summary.txt
