"""A whole BSA step captured into a CUDA graph (runner.BSAStepGraph) replays to the eager result."""
import pytest
import torch

import bsa_gen
from paper_2509_01085_b200 import Geometry

pytestmark = pytest.mark.gpu


def test_step_graph_replays_eager_result():
    from paper_2509_01085_b200.runner import BSAAttention, BSAStepGraph
    grid, Hh, d = (8, 12, 16), 2, 128
    g = Geometry(*grid)
    Q, K, V = bsa_gen.make_inputs("video", 4, 1, Hh, grid, d, device="cuda")
    dO = bsa_gen.grad_output(4, (1, Hh, g.L, d)).cuda()
    layer = BSAAttention(g, 0.5, 0.25, 0.9, 1, Hh, d, cache_partition=False)
    layer.forward(Q, K, V)
    ref = [x.clone() for x in (layer.O, *layer.backward(dO))]
    sg = BSAStepGraph(layer, Q, K, V, dO)
    # new inputs through the captured buffers: the replay must follow them
    Q2, K2, V2 = bsa_gen.make_inputs("video", 5, 1, Hh, grid, d, device="cuda")
    for dst, src in zip((Q, K, V), (Q2, K2, V2)):
        dst.copy_(src)
    out = [x.clone() for x in sg.replay()]
    torch.cuda.synchronize()
    eager = BSAAttention(g, 0.5, 0.25, 0.9, 1, Hh, d)
    eager.forward(Q2, K2, V2)
    want = [x.clone() for x in (eager.O, *eager.backward(dO))]
    torch.cuda.synchronize()
    assert torch.equal(out[0], want[0])  # forward: deterministic
    for a, b in zip(out[1:], want[1:]):  # dQ via fp32 reduce-adds: summation order only
        rms = b.float().pow(2).mean().sqrt().item()
        assert (a.float() - b.float()).abs().mean().item() <= 1e-3 * rms
    assert not torch.equal(out[0], ref[0])  # and it is not the first input's result
