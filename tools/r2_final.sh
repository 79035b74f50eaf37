mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "all rc=$?" >> gpurun_out/gputest.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
S=gpurun_out/solo_final.jsonl; rm -f $S
for n in 2 4 8; do
  timeout -s KILL 90 python bench.py --config b --solo $n --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $S
done
timeout -s KILL 400 python bench.py > gpurun_out/bench_d.log 2>&1
