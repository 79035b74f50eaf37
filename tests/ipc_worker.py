"""One rank of a multi-process RTP run on the IPC transport (spawned by
tests/test_gpu_ipc.py; all ranks may share GPU 0). Runs the golden RtpLinear
or MLP fixture on this rank's rows and saves its outputs to an .npz.

python tests/ipc_worker.py <case: linear|mlp|stack> <n> <rank> <uid hex> <mode> <out.npz>
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import to_dev, to_np  # noqa: E402
from paper_2311_01635_b200 import rtp  # noqa: E402


def main():
    case, n, rank, uid_hex, mode, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5], \
        sys.argv[6]
    dev = int(os.environ.get("RTPB_IPC_DEVICE", "0"))
    torch.cuda.set_device(dev)
    g = rtp.WorkerGroup.ipc(n, rank, dev, bytes.fromhex(uid_hex))
    fx = np.load(os.path.join(ROOT, "tests", "golden", f"{case}.npz")) if case != "stack" else None
    res = {}
    if case == "linear":
        w, b, x, dy = fx["w"], fx["b"], fx["x"], fx["dy"]
        M = x.shape[0] // n
        lin = rtp.RtpLinear(g, "lin", w.shape[0], w.shape[1], "bf16", weight=w, bias=b)
        lin.set_rotation_mode(mode)
        if mode == "outofplace":
            lin.allocate_comm_spares()
        lin.zero_grads()
        y = lin.forward([to_dev(x[rank * M:(rank + 1) * M], "bf16")])[0]
        res["fwd_id"] = lin.slot(rank)["logical_id"]
        dx = lin.backward([to_dev(dy[rank * M:(rank + 1) * M], "bf16")])[0]
        g.synchronize()
        led = g.ledger(rank)  # this process's device ledger (per-rank memory, not a simulation)
        res["ledger"] = np.array([led["peak_param"], led["peak_grad"], led["peak_comm"]], np.int64)
        res.update(y=to_np(y), dx=to_np(dx), grad=to_np(lin.grad_shard(rank)), weight=to_np(lin.weight_shard(rank)),
                   bwd_id=lin.slot(rank)["logical_id"], trace=np.array(lin.trace()),
                   traffic=np.array([[{"rotation_cw": 0, "rotation_ccw": 1}[k], a, c] for k, a, c in g.traffic()]))
        lin.close()
    elif case == "stack":
        from helpers import run_stack_local
        res.update(run_stack_local(g, [rank], n, chain=os.environ.get("RTPB_TEST_CHAIN", "1") == "1"))
    else:
        w1, b1, w2, b2, x, dy = (fx[k] for k in ("w1", "b1", "w2", "b2", "x", "dy"))
        M = x.shape[0] // n
        m = rtp.RtpMlp(g, "mlp", w1.shape[0], w1.shape[1], "bf16", w1=w1, b1=b1, w2=w2, b2=b2)
        m.set_rotation_mode(mode)
        m.begin_step()
        m.zero_grads()
        y = m.forward([to_dev(x[rank * M:(rank + 1) * M], "bf16")])[0]
        dx = m.backward([to_dev(dy[rank * M:(rank + 1) * M], "bf16")])[0]
        g.synchronize()
        res.update(y=to_np(y), dx=to_np(dx), grad1=to_np(m.ffn1.grad_shard(rank)), grad2=to_np(m.ffn2.grad_shard(rank)))
        m.close()
    g.close()
    np.savez(out, **res)


if __name__ == "__main__":
    main()
