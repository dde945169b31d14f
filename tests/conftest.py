import os
import sys

# The golden fixtures were generated with one OpenBLAS thread:
# OpenBLAS is not bitwise thread-invariant, so pin it before numpy loads.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

# In-process multi-rank emulation (parallel.run_threads with PeerComm) runs
# kernels that spin on each other's exchange signals from different streams
# of one device.  Streams that share a hardware work queue serialise, which
# would make a rank's spinning kernel block the very kernels it waits for;
# 32 connections give every rank stream its own queue.  (Ranks on different
# GPUs or in different processes never share a queue.)  Read at CUDA init.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
