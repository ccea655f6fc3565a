# K2 deep profile: one --set full capture (source-level stalls) of k_stage_nhwc_flat at the C2 micro shape
TAG=${TAG:-r02_k2_v6}
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_stage_nhwc" -c 2 -o gpurun_out/${TAG}_full python tools/profile_step.py > gpurun_out/${TAG}_full.out 2>&1
echo rc=$?
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>&1
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details > gpurun_out/${TAG}_details.txt 2>&1
ls -la gpurun_out/ | grep ${TAG}
