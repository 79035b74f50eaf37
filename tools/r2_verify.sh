mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "all rc=$?" >> gpurun_out/gputest.log
timeout -s KILL 400 python bench.py > gpurun_out/bench_d.log 2>&1
timeout -s KILL 120 python bench.py --config b --solo 8 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bench_b8.log 2>&1
timeout -s KILL 120 python bench.py --config b --solo 4 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bench_b4.log 2>&1
timeout -s KILL 120 python bench.py --config b --solo 2 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bench_b2.log 2>&1
