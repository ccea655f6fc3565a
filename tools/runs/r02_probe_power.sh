# clock / power of the no-stream baseline vs the MBS engine at 1 and 64 micro-batches per mini-batch (U-Net@384)
timeout 1200 python tools/probe_power.py --config n1 --seconds 45 > gpurun_out/ppw_n1.log 2> gpurun_out/ppw_n1.err; echo rc=$?; cat gpurun_out/ppw_n1.log; tail -3 gpurun_out/ppw_n1.err
