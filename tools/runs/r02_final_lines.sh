# final bench lines: C4 default (the driver's config) and N1, with the matched-weight-state baseline
timeout 1800 python bench.py > gpurun_out/fin_c4.json 2> gpurun_out/fin_c4.err; echo "c4 rc=$?"; tail -c 400 gpurun_out/fin_c4.json
timeout 3000 python bench.py --config n1 > gpurun_out/fin_n1.json 2> gpurun_out/fin_n1.err; echo "n1 rc=$?"; tail -c 400 gpurun_out/fin_n1.json
