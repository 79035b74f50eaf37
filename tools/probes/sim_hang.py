"""Dev probe: the simulated-ring stack (tests/sim_worker.py) with a watchdog
that dumps every worker's arrival flags / count-ins while it runs."""
import ctypes as C
import os
import sys
import threading
import time

os.environ.setdefault("RTPB_FLAGS", "1")
os.environ.setdefault("RTPB_SIM_FLAGS", "1")
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from helpers import run_stack_local  # noqa: E402
from paper_2311_01635_b200 import _lib, rtp  # noqa: E402

import torch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
PIN = torch.zeros(128, dtype=torch.int32, pin_memory=True)  # pinned before any work
g = rtp.WorkerGroup(n, "lockstep")
state = {"done": False, "err": None}


def work():
    try:
        run_stack_local(g, list(range(n)), n, chain=True)
    except Exception as e:  # noqa: BLE001
        state["err"] = repr(e)
    state["done"] = True


for r in range(n):
    print(f"worker {r} flag pool at 0x{_lib.lib.rtpb_debug_flag_address(g._h, r, 0):x} (128 per layer: F 0, W 16, G 32, "
          f"doneF 64, doneB 80, doneW 96)", flush=True)
_busy = C.c_int()
_lib.lib.rtpb_debug_read_flags(g._h, 0, 0, 128, C.cast(PIN.data_ptr(), C.POINTER(C.c_uint)), C.byref(_busy))
t = threading.Thread(target=work, daemon=True)
t.start()
for i in range(4):
    time.sleep(3.0)
    if state["done"]:
        break
    for layer in range(2):
        line = []
        for r in range(n):
            busy = C.c_int()
            rc = _lib.lib.rtpb_debug_read_flags(g._h, r, layer * 128, 128, C.cast(PIN.data_ptr(), C.POINTER(C.c_uint)),
                                                C.byref(busy))
            v = PIN.tolist()
            line.append(f"r{r} rc{rc} b{busy.value} F{v[0:n]} W{v[16:16 + n]} G{v[32:32 + n]} dF{v[64:64 + n]} dB{v[80:80 + n]} "
                        f"dW{v[96:96 + n]}")
        print(f"t={3 * (i + 1)}s L{layer}: " + " | ".join(line), flush=True)
print("done:", state, flush=True)
os._exit(0)
