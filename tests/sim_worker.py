"""Runs the 3-block chained stack (helpers.run_stack_local) on an in-process
Lockstep group of n workers sharing GPU 0 and saves every output to an .npz.
Spawned by tests/test_gpu_pass.py with and without RTPB_FLAGS=1
RTPB_SIM_FLAGS=1 (the arrival-flag / pass-launch protocol with each worker's
grids on its share of the SMs), since both switches are read once per process.

python tests/sim_worker.py <n> <out.npz>
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import run_stack_local  # noqa: E402
from paper_2311_01635_b200 import rtp  # noqa: E402


def main():
    n, out = int(sys.argv[1]), sys.argv[2]
    g = rtp.WorkerGroup(n, "lockstep")
    res = run_stack_local(g, list(range(n)), n, chain=True)
    g.close()
    np.savez(out, **res)


if __name__ == "__main__":
    main()
