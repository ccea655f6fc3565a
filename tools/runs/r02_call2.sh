# changed GPU tests, compute-sanitizer pass, ncu launch list + full capture of the MBS kernels
TAG=${TAG:-r02_c2_v2}
timeout 900 python -m pytest tests/test_bn_gpu.py tests/test_pool_gpu.py tests/test_cli_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/c2_tests.log 2>&1; echo rc=$? >> gpurun_out/c2_tests.log; tail -5 gpurun_out/c2_tests.log
TAG=$TAG bash tools/runs/r02_profile.sh
bash tools/runs/r02_sanitize.sh
