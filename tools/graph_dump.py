#!/usr/bin/env python
"""Capture three gemm() calls into a CUDA graph and write its DOT description
(node types, kernel launch attributes, edge types) to gpurun_out/gd/graph.dot."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from cuda.bindings import runtime as rt
import paper_2407_10960_b200 as F
m, k, n, bits, group = 1, 4096, 14336, 3, 128
rng = np.random.default_rng(0)
idx, sc = F.quantize_matrix(rng.standard_normal((k, n), dtype=np.float32), bits, group)
dws = [F.DeviceWeights(idx, sc, F.build_nf_table(bits), bits, group) for _ in range(3)]
x = torch.randn(m, k, dtype=torch.float16, device="cuda")
y = torch.empty(m, n, dtype=torch.float16, device="cuda")
st = torch.cuda.Stream()
for d in dws:
    d.gemm(x, y, stream=st.cuda_stream)
st.synchronize()
err, = rt.cudaStreamBeginCapture(st.cuda_stream, rt.cudaStreamCaptureMode.cudaStreamCaptureModeGlobal)
for d in dws:
    d.gemm(x, y, stream=st.cuda_stream)
err, graph = rt.cudaStreamEndCapture(st.cuda_stream)
print("capture", err)
os.makedirs("gpurun_out/gd", exist_ok=True)
print(rt.cudaGraphDebugDotPrint(graph, b"gpurun_out/gd/graph.dot", 0xFFFF))
