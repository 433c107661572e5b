"""B200-native (sm_100a) VecAttention hot path: important-vector selection +
vector-sparse attention behind a C ABI (include/vecattn.h).

The CUDA library is loaded lazily by ``paper_2603_29494_b200.vecattn.load()``;
importing the package does not touch the GPU.
"""
__all__ = ["vecattn", "synth"]
