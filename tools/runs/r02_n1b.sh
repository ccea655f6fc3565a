# N1 with the no-stream baseline as long as the e2e run; then the K2 warp-specialised sanitizer pass
timeout 3000 python bench.py --config n1 --steps 3 --warmup 3 > gpurun_out/n1b_bench.json 2> gpurun_out/n1b_bench.err; echo "rc=$?"
tail -c 600 gpurun_out/n1b_bench.json
bash tools/runs/r02_sanitize_k2ws.sh
