"""Small workloads for compute-sanitizer (tools/sanitize.sh): every in-kernel
protocol of the step GEMMs at shapes small enough for racecheck.

  fused   N = 1 MLP: the scheduled two-problem forward (row-block counters,
          done_ctas reset) and the concurrent D / W backward launches (dpre
          row-block waits across launches)
  splitk  one rank of an 8-way ring (solo) at config (b)'s thin shard shapes:
          dW split-K ordered chains and slice folds, paired dX, bias tickets
  flags   the same with shard-arrival flags (RTPB_FLAGS=1: in-kernel flag
          waits, the last reader grid's flag reset)
  f32     N = 4 RtpLinear in fp32 mode (3xTF32 operand splits)
Usage: python tools/sanitize_driver.py <case> [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01635_b200 import rtp  # noqa: E402


def mlp_steps(grp, h, f, M, steps, dtype="bf16"):
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    m = rtp.RtpMlp(grp, "san", h, f, dtype, seed=42, stream_base=0)
    m.set_rotation_mode("outofplace")
    m.begin_step()
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [(torch.rand(M, h, device="cuda", generator=g) * 2 - 1).to(tdt) for _ in grp.local_ranks]
    dys = [(torch.rand(M, h, device="cuda", generator=g) * 2 - 1).to(tdt) for _ in grp.local_ranks]
    for _ in range(steps):
        m.zero_grads()
        m.forward(xs)
        m.backward(dys)
    grp.synchronize()
    m.close()


def main():
    case = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    torch.cuda.set_device(0)
    if case == "fused":
        mlp_steps(rtp.WorkerGroup(1), 256, 1024, 512, steps)
    elif case in ("splitk", "flags"):
        mlp_steps(rtp.WorkerGroup.solo(8, 0, 0), 768, 3072, 1024, steps)
    elif case == "f32":
        g = rtp.WorkerGroup(4)
        lin = rtp.RtpLinear(g, "lin", 128, 256, "f32", seed=1, stream_base=0)
        xs = [torch.rand(64, 128, device="cuda") for _ in range(4)]
        dys = [torch.rand(64, 256, device="cuda") for _ in range(4)]
        for _ in range(steps):
            lin.zero_grads()
            lin.forward(xs)
            lin.backward(dys)
        g.synchronize()
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(f"sanitize case {case}: ok")


if __name__ == "__main__":
    main()
