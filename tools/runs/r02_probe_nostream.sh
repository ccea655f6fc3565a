# no-stream baseline data A/B (two cycled batches vs 64 distinct batches), U-Net@384 and ResNet-50@224
timeout 900 python tools/probe_nostream_data.py --config n1 --seconds 60 > gpurun_out/pns_n1.log 2> gpurun_out/pns_n1.err; echo rc=$?; cat gpurun_out/pns_n1.log
timeout 600 python tools/probe_nostream_data.py --config c2 --seconds 40 > gpurun_out/pns_c2.log 2> gpurun_out/pns_c2.err; echo rc=$?; cat gpurun_out/pns_c2.log
