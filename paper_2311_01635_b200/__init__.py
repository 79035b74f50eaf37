"""B200-native Rotated Tensor Parallelism (arXiv 2311.01635) hot path.

The RTP linear / MLP forward+backward over a ring of workers, as sm_100a
tcgen05 step kernels + a C++ host runtime (librtpb.so, include/rtpb.h).
`paper_2311_01635_b200.rtp` mirrors the reference's layer API.
"""
import os as _os

# A worker drives three streams (compute, comm, aux); with CUDA's default of 8
# hardware work queues per device, streams share queues, and work queued
# behind a comm stream's memory wait waits with it. More queues keep the
# workers' streams apart (read when CUDA initialises; a caller's own setting wins).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import _lib  # noqa: E402,F401  (fails loudly if the native library is missing)
