mkdir -p gpurun_out
O=gpurun_out/wgrad_ab.txt; rm -f $O
for v in default nocolsum; do
  if [ $v = default ]; then unset RTPB_LIB; else export RTPB_LIB=build/var_nocolsum/librtpb.so; fi
  echo "== $v" >> $O
  for s in "16384 4096 16384" "16384 16384 4096" "16384 4096 2048" "16384 16384 512"; do
    timeout -s KILL 120 python tools/gemm_one.py $s fwd,dgrad,wgrad,wgrad_as_dgrad >> $O 2>&1
  done
done
