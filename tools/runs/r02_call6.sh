# final-state: accum/stage/engine GPU tests, default bench (C4) + reference arm, launch list and --set full
TAG=${TAG:-r02_c2_v5}
timeout 900 python -m pytest tests/test_accum_gpu.py tests/test_engine_gpu.py tests/test_optim_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/c6_tests.log 2>&1; echo rc=$? >> gpurun_out/c6_tests.log; tail -3 gpurun_out/c6_tests.log
timeout 1800 python bench.py > gpurun_out/c6_bench.json 2> gpurun_out/c6_bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/c6_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/c6_ref.json 2> gpurun_out/c6_ref.err; echo "ref rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py > gpurun_out/${TAG}_launches.out 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_stage|k_accum|k_finalize|k_sgd|k_gather" -o gpurun_out/${TAG}_full python tools/profile_step.py > gpurun_out/${TAG}_full.out 2>&1
ls -la gpurun_out | grep $TAG
