# round-2 re-entry check: full GPU suite, smoke, default bench line (C4), reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/chk_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/chk_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/chk_pytest_gpu.log; tail -15 gpurun_out/chk_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; tail -3 gpurun_out/chk_smoke.log
timeout 1800 python bench.py > gpurun_out/chk_bench.json 2> gpurun_out/chk_bench.err; tail -c 3000 gpurun_out/chk_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/chk_ref.json 2> gpurun_out/chk_ref.err; cat gpurun_out/chk_ref.json
