# K2 conversion change: staging parity tests, kbench, ncu of the K2 launches; then the N1 bench line and
# a 2-rank (gloo, one GPU) bench.py run
timeout 600 python -m pytest tests/test_stage_gpu.py tests/test_tracer_gpu.py tests/test_fullsize_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/c3_tests.log 2>&1; echo rc=$? >> gpurun_out/c3_tests.log; tail -3 gpurun_out/c3_tests.log
timeout 300 python tools/kbench.py --config c2 > gpurun_out/c3_kbench_c2.json 2>&1; grep -A5 k2_ gpurun_out/c3_kbench_c2.json | grep -E "k2_|us_median|frac"
timeout 300 python tools/kbench.py --config c3 > gpurun_out/c3_kbench_c3.json 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_stage|k_accum" -c 6 -o gpurun_out/r02_c2_v3_k2 python tools/profile_step.py > gpurun_out/r02_c2_v3_k2.out 2>&1
timeout 2400 python bench.py --config n1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/n1_bench.json 2> gpurun_out/n1_bench.err; echo "n1 rc=$?"; tail -c 1500 gpurun_out/n1_bench.json
MBS_DP_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --no-fp32-context > gpurun_out/dp2_gloo_bench.json 2> gpurun_out/dp2_gloo_bench.err; echo "dp2 rc=$?"; tail -c 1500 gpurun_out/dp2_gloo_bench.json
