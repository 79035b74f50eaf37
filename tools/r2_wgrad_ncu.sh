mkdir -p gpurun_out
for k in wgrad wgrad_as_dgrad dgrad; do
  timeout -s KILL 300 ncu --set full --clock-control none -k regex:rtp_gemm -s 3 -c 1 -o gpurun_out/w_$k \
     python tools/gemm_one.py 16384 4096 16384 $k > gpurun_out/w_$k.log 2>&1
  ncu -i gpurun_out/w_$k.ncu-rep --page raw --csv > gpurun_out/w_raw_$k.csv 2>/dev/null
  ncu -i gpurun_out/w_$k.ncu-rep --page details --csv > gpurun_out/w_det_$k.csv 2>/dev/null
  rm -f gpurun_out/w_$k.ncu-rep
done
