# full GPU suite + smoke + default bench (C4) + reference arm with the final bench.py
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/c13_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/c13_pytest_gpu.log; tail -4 gpurun_out/c13_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c13_smoke.log 2>&1; tail -3 gpurun_out/c13_smoke.log
timeout 2400 python bench.py --steps 5 --warmup 3 > gpurun_out/c13_bench.json 2> gpurun_out/c13_bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/c13_bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/c13_ref.json 2> gpurun_out/c13_ref.err; echo "ref rc=$?"
