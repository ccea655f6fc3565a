# is it the weights' trajectory? the MBS engine at one micro-batch per step with lr 0 vs lr 0.01, and 64 micros
timeout 1200 python tools/probe_power.py --config n1 --seconds 45 --kinds mbs_1_lr0,mbs_1,mbs_64 --reps 1 > gpurun_out/ppw2_n1.log 2> gpurun_out/ppw2_n1.err; echo rc=$?; cat gpurun_out/ppw2_n1.log; tail -3 gpurun_out/ppw2_n1.err
