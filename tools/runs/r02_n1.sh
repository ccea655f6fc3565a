# N1 (U-Net@384, 80,000 host samples > HBM as fp32) with the final bench.py (>= 30 s no-stream run, per-clock ratio)
timeout 3000 python bench.py --config n1 --steps 3 --warmup 3 > gpurun_out/n1_bench.json 2> gpurun_out/n1_bench.err; echo "rc=$?"
tail -c 1500 gpurun_out/n1_bench.json
