# final GPU suite + smoke with the final tree
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fs_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/fs_pytest_gpu.log; tail -4 gpurun_out/fs_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fs_smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/fs_smoke.log
