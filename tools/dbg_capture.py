"""Debug (not product): find the first op that invalidates a frame-graph
capture, replaying the failing test order (cascades, 1-rank NCCL exchange,
two-shard C2)."""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import runtime as rt
from paper_2511_02852_b200 import _native as N

cap = {"s": None, "bad": False}
real_call = N.call


def status():
    s = cap["s"]
    if s is None:
        return None
    err, st, *_ = rt.cudaStreamGetCaptureInfo(s.cuda_stream)
    return st


def spy(name, a, stream):
    before = status()
    real_call(name, a, stream)
    after = status()
    if after is not None and not cap["bad"] and after != rt.cudaStreamCaptureStatus.cudaStreamCaptureStatusActive:
        cap["bad"] = True
        print("capture invalid after", name, before, after, flush=True)
N.call = spy
from paper_2511_02852_b200 import harness as H
real_cs = H.Simulation._capture_stream
def cs(self):
    s = real_cs(self)
    cap["s"] = s
    cap["bad"] = False
    print("capture stream", hex(s.cuda_stream), flush=True)
    return s
H.Simulation._capture_stream = cs
real_side = H.Simulation._side_stream
def side(self, name="fft"):
    s = real_side(self, name)
    return s
H.Simulation._side_stream = side

import pytest
sys.exit(pytest.main(["-q", "-x", "-s", "-m", "gpu", "tests/test_gpu_cascades.py", "tests/test_gpu_exchange.py"]))
