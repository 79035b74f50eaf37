"""B200-native Rotated Tensor Parallelism (arXiv 2311.01635) hot path.

The RTP linear / MLP forward+backward over a ring of workers, as sm_100a
tcgen05 step kernels + a C++ host runtime (librtpb.so, include/rtpb.h).
`paper_2311_01635_b200.rtp` mirrors the reference's layer API.
"""
from . import _lib  # noqa: F401  (fails loudly if the native library is missing)
