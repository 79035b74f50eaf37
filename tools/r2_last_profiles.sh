mkdir -p gpurun_out
# config (d) N = 1 (the bench default): launch list + full capture of 3 step GEMMs
LAUNCH_CAP=800 bash tools/profile_round.sh r2e 40 3
# synccheck / racecheck over the pass launches (flags preset; no cross-stream waits)
timeout -s KILL 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_pass.py -x -q -p no:cacheprovider -k "fwd_pass_equals or dgrad_pass_equals or paired" > gpurun_out/synccheck_pass.log 2>&1; echo "rc=$?" >> gpurun_out/synccheck_pass.log
