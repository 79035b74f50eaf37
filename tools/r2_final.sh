mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "all rc=$?" >> gpurun_out/gputest.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 400 python bench.py > gpurun_out/bench_d.log 2>&1
