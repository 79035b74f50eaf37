import torch
try:
    from cuda.bindings import driver as cu
except ImportError:
    from cuda import cuda as cu
torch.cuda.init()
buf = torch.zeros(4, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
side = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    g.capture_begin()
    ev = torch.cuda.Event(); ev.record(s); side.wait_event(ev)
    r = cu.cuStreamWriteValue32(side.cuda_stream, buf.data_ptr(), 7, 0)
    print("write in capture:", r)
    r = cu.cuStreamWaitValue32(s.cuda_stream, buf.data_ptr(), 7, cu.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ)
    print("wait in capture:", r)
    ev2 = torch.cuda.Event(); ev2.record(side); s.wait_event(ev2)
    buf.add_(1)
    g.capture_end()
g.replay(); torch.cuda.synchronize(); print(buf.tolist())
