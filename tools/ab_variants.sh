for v in default nocolsum promo128; do
  if [ $v = default ]; then unset RTPB_LIB; else export RTPB_LIB=build/var_$v/librtpb.so; fi
  echo "== $v"
  for s in "16384 4096 4096" "8192 3072 768" "8192 768 3072"; do python tools/gemm_one.py $s fwd,dgrad,wgrad 2>&1 | grep -v Warn; done
done
