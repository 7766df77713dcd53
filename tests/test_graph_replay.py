"""CUDA-graph replays with changing inputs: the refresh kernel's in-kernel
split merge (C2 b=16 shape: items span 2 CTAs) must see the current replay's
partials, never a previous replay's (its ready flags are reset by every
launch).  Compared against eager launches on the same inputs."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_refresh_graph_replays_track_new_inputs():
    from paper_2602_05305_b200 import kernels as K

    groups, n, d = 128, 32768, 128  # C2 b=16
    g = torch.Generator(device="cuda").manual_seed(9)
    q = torch.randn((groups, 128, d), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((groups, n, d), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((groups, n, d), device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty((groups, 128, d), device="cuda", dtype=torch.float32)
    l = torch.empty((groups, 128), device="cuda", dtype=torch.float32)
    s = torch.cuda.Stream()
    K.attention_partial(q, k, v, 0, n, None, o, l)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        K.attention_partial(q, k, v, 0, n, None, o, l)
    for it in range(4):
        # new inputs in place, then replay; compare with an eager launch
        q.copy_(torch.randn(q.shape, device="cuda", generator=g).to(torch.bfloat16))
        v.mul_(-1.0)
        gr.replay()
        torch.cuda.synchronize()
        oe, le = K.attention_partial(q, k, v)
        torch.cuda.synchronize()
        assert torch.equal(o, oe) and torch.equal(l, le), f"replay {it} differs from eager"
