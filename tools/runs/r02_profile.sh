# round-2 profiling pass: changed GPU tests, launch list + one --set full capture of the MBS kernels (C2 micro shape)
TAG=${TAG:-r02_c2_v1}
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_tracer_gpu.py tests/test_paper_parity_gpu.py tests/test_stem_gpu.py -q -m gpu -p no:cacheprovider -s > gpurun_out/t_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/t_${TAG}.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py > gpurun_out/${TAG}_launches.out 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_stage|k_accum|k_finalize|k_sgd|k_gather" -o gpurun_out/${TAG}_full python tools/profile_step.py > gpurun_out/${TAG}_full.out 2>&1
ls -la gpurun_out/ | grep ${TAG}
