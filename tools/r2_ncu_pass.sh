mkdir -p gpurun_out
# the forward and dX pass launches of config (b) at N = 8 (Solo, flags raised up front for the serial profiler)
RTPB_SERIAL_PROFILE=1 timeout -s KILL 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
   -k 'regex:GemmCfg<\(int\)[01],' -s 4 -c 4 -o gpurun_out/full_r2c python tools/pass_ncu_probe.py > gpurun_out/ncu_full_r2c.log 2>&1
ncu -i gpurun_out/full_r2c.ncu-rep --page raw --csv > gpurun_out/full_raw_r2c.csv 2>/dev/null
ncu -i gpurun_out/full_r2c.ncu-rep --page source --csv --print-source sass > gpurun_out/full_src_r2c.csv 2>/dev/null
