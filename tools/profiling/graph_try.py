"""Does a whole BSA step (selection + fwd + bwd through the C ABI) capture into a CUDA graph, and what does
replay save over eager launches? python tools/profiling/graph_try.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402
from paper_2509_01085_b200.runner import BSAAttention  # noqa: E402

g = bsa.Geometry(21, 30, 52)
Q, K, V = bsa_gen.make_inputs("video", 0, 1, 12, (21, 30, 52), 128, device="cuda")
dO = bsa_gen.grad_output(0, (1, 12, g.L, 128)).cuda()
layer = BSAAttention(g, 0.5, 0.1, 0.9, 1, 12, 128, cache_partition=False)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        layer.forward(Q, K, V)
        layer.backward(dO)
torch.cuda.synchronize()
O_ref, dQ_ref = layer.O.clone(), layer.dQ.clone()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=s):
    layer.forward(Q, K, V)
    layer.backward(dO)
torch.cuda.synchronize()


def t(fn, n=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def eager():
    layer.forward(Q, K, V)
    layer.backward(dO)


print("eager ms", t(eager), "graph ms", t(graph.replay))
graph.replay()
torch.cuda.synchronize()
print("O equal after replay:", torch.equal(layer.O, O_ref), " dQ max diff:", (layer.dQ.float() - dQ_ref.float()).abs().max().item())
