mkdir -p gpurun_out
GRAPH=1 SOLO=8 RTPB_FLAGS=1 timeout -s KILL 120 python tools/timeline.py > gpurun_out/tl_b8_pass.txt 2>&1
RTPB_FLAGS=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launch_d8_pass.csv python tools/rtp_sweep.py --config d --solo 8 --blocks 1 --steps 1 --warmup 1 > gpurun_out/launch_d8_pass.log 2>&1
# IPC n=4 MLP with pass launches, long timeout: slow or stuck?
python - > gpurun_out/ipc4.txt 2>&1 <<'PY'
import os, subprocess, sys, time
sys.path.insert(0, ".")
from paper_2311_01635_b200 import rtp
for env in ({"RTPB_FLAGS": "1", "RTPB_NO_PASS": "1"}, {"RTPB_FLAGS": "1"}):
    uid = rtp.WorkerGroup.ipc_unique_id().hex()
    t0 = time.time()
    ps = [subprocess.Popen([sys.executable, "tests/ipc_worker.py", "mlp", "4", str(r), uid, "outofplace", f"/tmp/o{r}.npz"],
                           stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env={**os.environ, **env}) for r in range(4)]
    for p in ps:
        try:
            out = p.communicate(timeout=400)[0]
            print(env, "rc", p.returncode, "t", round(time.time() - t0, 1), out[-500:], flush=True)
        except subprocess.TimeoutExpired:
            print(env, "TIMEOUT", flush=True)
            for q in ps: q.kill()
            break
PY
