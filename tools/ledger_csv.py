"""The reference's memory reports (`rtpsim ledger` / `rtpsim sweep`,
proj/src/commands.cpp:112-143 and 165-181) from the DEVICE ledger: same CSV
schemas and column order, the peaks being bytes of B200 memory per worker for
an RTP MLP block (bf16 weights, fp32 gradients), N workers simulated on GPU 0.

  ledger: strategy,n,category,peak_bytes,duplication
          (duplication = n * peak - serial peak, analysis.cpp:335-340)
  sweep:  strategy,n,batch_per_worker,global_batch,param_peak,grad_peak,
          activation_peak,commbuffer_peak,other_peak,total_peak

python tools/ledger_csv.py [--h 768 --f 3072 --n 4 --rows 1024] [--sweep 256,512,1024]
"""
from __future__ import annotations

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01635_b200 import reports, rtp  # noqa: E402

CATS = ("Param", "Grad", "Activation", "CommBuffer", "Other")
KEYS = ("param", "grad", "activation", "comm", "other")


def run(n, mode, rows_per_worker, h, f):
    """One fwd+bwd step of an RTP MLP; returns the worst worker's peaks."""
    grp = rtp.WorkerGroup(n, "lockstep", devices=[0] * n)
    grp.reset_ledger_peaks()
    mlp = rtp.RtpMlp(grp, "mlp", h, f, "bf16", seed=42, stream_base=0)
    mlp.set_rotation_mode(mode)
    mlp.begin_step()
    mlp.zero_grads()
    g = torch.Generator(device="cuda").manual_seed(42)
    xs = [(torch.rand(rows_per_worker, h, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(n)]
    dys = [(torch.rand(rows_per_worker, h, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(n)]
    mlp.forward(xs)
    mlp.backward(dys)
    grp.synchronize()
    led = [grp.ledger(r) for r in range(n)]
    worst = max(led, key=lambda d: d["peak_total"])
    out = {c: worst["peak_" + k] for c, k in zip(CATS, KEYS)}
    out["total"] = worst["peak_total"]
    mlp.close()
    grp.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--h", type=int, default=768)
    ap.add_argument("--f", type=int, default=3072)
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--rows", type=int, default=1024, help="global batch rows for the ledger report")
    ap.add_argument("--sweep", default="256,512,1024", help="rows per worker for the sweep report")
    ap.add_argument("--out", default=None, help="directory for ledger.csv / sweep.csv (default: stdout)")
    args = ap.parse_args()
    torch.cuda.set_device(0)

    serial = run(1, "inplace", args.rows, args.h, args.f)
    runs = [("serial", 1, serial)]
    for strat, mode in (("rtp-inplace", "inplace"), ("rtp-outofplace", "outofplace")):
        runs.append((strat, args.n, run(args.n, mode, args.rows // args.n, args.h, args.f)))
    ledger = reports.ledger_csv(serial, runs[1:])
    sweep = ""
    for strat, mode in (("rtp-inplace", "inplace"), ("rtp-outofplace", "outofplace")):
        pts = []
        for b in (int(v) for v in args.sweep.split(",")):
            pk = run(args.n, mode, b, args.h, args.f)
            pts.append((b, pk, pk["total"]))
        text = reports.sweep_csv(strat, args.n, pts)
        sweep += text if not sweep else text.split("\n", 1)[1]
    if args.out:
        os.makedirs(args.out, exist_ok=True)
        open(os.path.join(args.out, "ledger.csv"), "w").write(ledger)
        open(os.path.join(args.out, "sweep.csv"), "w").write(sweep)
    print(ledger + "\n" + sweep, end="")


if __name__ == "__main__":
    main()
