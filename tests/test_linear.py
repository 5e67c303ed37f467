"""MackoLinear (nn.Linear replacement for batch-1 decode) on cuda:0 against the oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2511_13061_b200 import macko as M
from paper_2511_13061_b200.linear import MackoLinear
from tests.helpers import b200_y, to_dev, to_host_u16

pytestmark = pytest.mark.gpu


def test_macko_linear_matches_oracle(cuda):
    out_f, in_f = 700, 3000
    A = O.gen_dense(out_f, in_f, 0.5, 81)
    lin = torch.nn.Linear(in_f, out_f, bias=True, device=cuda, dtype=torch.float16)
    with torch.no_grad():
        lin.weight.copy_(to_dev(A))
        lin.bias.uniform_(-1, 1)
    ml = MackoLinear.from_linear(lin)
    x = O.gen_vector(in_f, 82)
    xd = to_dev(x)
    y = ml(xd)
    torch.cuda.synchronize()
    y_ref = b200_y(O.encode_dense(A), x)
    expect = (torch.from_numpy(y_ref.view(np.float16)).to(cuda) + lin.bias).view(torch.int16)
    assert np.array_equal(to_host_u16(y), expect.cpu().numpy().view(np.uint16))
    # [1, 1, in] and a batch of 3 (one SpMV per vector)
    assert ml(xd.view(1, 1, -1)).shape == (1, 1, out_f)
    xb = torch.stack([xd, xd * 2, -xd])
    yb = ml(xb)
    assert yb.shape == (3, out_f)
    assert torch.equal(yb[0], y)
    with pytest.raises(ValueError):
        ml(torch.zeros(in_f + 1, dtype=torch.float16, device=cuda))


def test_torch_op_and_graph_capture(cuda):
    # torch.ops.macko.spmv: the registered operator, its fake (meta) kernel, and CUDA-graph capture
    out_f, in_f = 1000, 2048
    A = O.gen_dense(out_f, in_f, 0.5, 91)
    ml = MackoLinear(M.DeviceMatrix.from_dense(to_dev(A)))
    x = to_dev(O.gen_vector(in_f, 92))
    y = torch.ops.macko.spmv(ml.matrix.handle, x, out_f)
    torch.cuda.synchronize()
    assert np.array_equal(to_host_u16(y), b200_y(O.encode_dense(A), O.gen_vector(in_f, 92)))
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode() as mode:
        fx = mode.from_tensor(x)
        assert torch.ops.macko.spmv(ml.matrix.handle, fx, out_f).shape == (out_f,)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ml(x)  # warm-up outside capture
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        yg = ml(x)
    x.copy_(to_dev(O.gen_vector(in_f, 93)))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(yg, ml(x))
    with pytest.raises(ValueError):
        torch.ops.macko.spmv(ml.matrix.handle, x.float(), out_f)
