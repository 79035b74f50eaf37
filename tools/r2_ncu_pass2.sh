mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_pass.py -x -q -p no:cacheprovider > gpurun_out/pass.log 2>&1; echo "rc=$?" >> gpurun_out/pass.log
bash tools/r2_ncu_pass.sh
# the dW pass too, now that steps never share a split-K chain counter
RTPB_SERIAL_PROFILE=1 timeout -s KILL 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
   -k 'regex:GemmCfg<\(int\)2,' -s 2 -c 2 -o gpurun_out/full_r2d python tools/pass_ncu_probe.py > gpurun_out/ncu_full_r2d.log 2>&1
ncu -i gpurun_out/full_r2d.ncu-rep --page raw --csv > gpurun_out/full_raw_r2d.csv 2>/dev/null
ncu -i gpurun_out/full_r2d.ncu-rep --page source --csv --print-source sass > gpurun_out/full_src_r2d.csv 2>/dev/null
