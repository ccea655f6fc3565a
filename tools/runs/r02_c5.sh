timeout 2400 python bench.py --config c5 > gpurun_out/fo2_c5.json 2> gpurun_out/fo2_c5.err; echo "c5 rc=$?"; tail -c 300 gpurun_out/fo2_c5.json; grep -c OutOfMemory gpurun_out/fo2_c5.err
