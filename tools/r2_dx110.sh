mkdir -p gpurun_out
for d in 110 124; do
RTPB_FLAGS=1 RTPB_PASS_DX_SMS=$d timeout -s KILL 90 python bench.py --config b --solo 8 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/dx$d.txt 2>&1
echo "rc=$?" >> gpurun_out/dx$d.txt
done
