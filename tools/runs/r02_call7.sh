# C4 (the driver's default config) through torchrun with 2 ranks sharing one GPU (gloo): the N>1 bench path at
# batch > HBM, with the shared host image pool
df -h /dev/shm /tmp | tee gpurun_out/c7_df.txt; free -g | tee -a gpurun_out/c7_df.txt; nproc >> gpurun_out/c7_df.txt
MBS_DP_BACKEND=gloo timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
    bench.py --gpus 2 --steps 1 --warmup 3 > gpurun_out/c7_dp2_c4.json 2> gpurun_out/c7_dp2_c4.err; echo "dp2 c4 rc=$?"; tail -c 800 gpurun_out/c7_dp2_c4.json; tail -5 gpurun_out/c7_dp2_c4.err
