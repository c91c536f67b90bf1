"""B200-native stall-free hybrid-batch forward (Sarathi-Serve hot path).

host  -- the reference scheduler/engine API over libss_host.so (C++20)
gpu   -- the ss_gpu.h boundary over libss_gpu.so (sm_100a kernels)
"""
__all__ = ["host", "gpu"]
