"""compute-sanitizer driver: small cases of every kernel — SpMV at every width, SpMM batches,
the dense and CSR compressors, csr_from_dense / dense_from_macko / padding_count, the device plan,
the host-buffer path, the fused all-gather instance (one local stand-in peer), a PDL decode chain and a small Llama decode step — checked against the
oracle (tools only).  Run: compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2511_13061_b200 import decoder_chain as D  # noqa: E402
from paper_2511_13061_b200 import llama as L  # noqa: E402
from paper_2511_13061_b200 import macko as M  # noqa: E402
from tests.helpers import b200_y, to_dev, to_host_u16  # noqa: E402

bad = 0
for bits in (1, 2, 4, 8):
    for R, C, d in ((37, 1000, 0.3), (300, 2500, 0.9), (5, 9000, 0.05), (8, 40000, 0.5)):  # last: split rows
        A = O.gen_dense(R, C, d, R + C + bits)
        x = O.gen_vector(C, 3)
        m = O.encode_dense(A, bits)
        dm = M.DeviceMatrix.from_dense(to_dev(A), b_delta=bits)
        h = dm.download()
        bad += int(not np.array_equal(h.values, m.values))
        y = to_host_u16(M.spmv(dm, to_dev(x)))
        bad += int(not np.array_equal(y, b200_y(m, x)))
        yp = torch.empty(R, dtype=torch.float16, device="cuda")  # the PDL (chain) kernel instance
        dm.spmv_into(to_dev(x), yp, pdl=True)
        torch.cuda.synchronize()
        bad += int(not np.array_equal(to_host_u16(yp), y))
        other = torch.full((R,), -1.0, dtype=torch.float16, device="cuda")  # the peers instance
        fl = torch.zeros(2, dtype=torch.int32, device="cuda")
        dm.set_peers([yp.data_ptr(), other.data_ptr()], [fl.data_ptr(), fl.data_ptr() + 4])
        dm.spmv_into(to_dev(x), yp, peers=True)
        torch.cuda.synchronize()
        bad += int(not np.array_equal(to_host_u16(other), y)) + int(not np.array_equal(to_host_u16(yp), y))
        dm.set_peers([], [])
        vals, cols, rp = M.csr_from_dense(A)
        dc = M.DeviceMatrix.from_csr(vals, cols, rp, R, C, bits)
        bad += int(not np.array_equal(dc.download().packed_deltas, m.deltas))
        bad += int(not np.array_equal(dc.to_dense(), A))
        bad += int(dc.padding_count() != O.padding_count(m))
        if bits == 4:
            X = np.stack([O.gen_vector(C, 10 + b) for b in range(5)])
            Y = torch.empty((5, R), dtype=torch.float16, device="cuda")
            dm.spmm_into(to_dev(X), Y)
            Yh = to_host_u16(Y)
            bad += sum(int(not np.array_equal(Yh[b], b200_y(m, X[b]))) for b in range(5))
        dm.close()
        dc.close()
A = O.gen_dense(200, 700, 0.5, 1)
dm = M.DeviceMatrix.from_dense(to_dev(A))
x = O.gen_vector(700, 2)
hx = torch.empty(700, dtype=torch.int16, pin_memory=True)
hx.numpy().view(np.uint16)[:] = x
hy = torch.zeros(200, dtype=torch.int16, pin_memory=True)
dm.spmv_host(hx.numpy().view(np.uint16), hy.numpy().view(np.uint16))
bad += int(not np.array_equal(hy.numpy().view(np.uint16), b200_y(O.encode_dense(A), x)))
ch = D.SparseDecoderChain(D.ChainShape(2, 256, 688), density=0.5, seed=3)
M.gen_vector(ch.acts["h"], 256, seed=4)
ch.acts["h"].mul_(2.0**-8)
h0 = ch.acts["h"].clone()
ch.forward_token(pdl=False)
torch.cuda.synchronize()
ref = to_host_u16(ch.acts["h"])
ch.acts["h"].copy_(h0)
ch.forward_token(pdl=True)
torch.cuda.synchronize()
bad += int(not np.array_equal(to_host_u16(ch.acts["h"]), ref))
w = L.LlamaWeights(L.LlamaConfig(vocab=500, hidden=256, layers=2, heads=2, inter=688, max_len=16), density=0.5)
dec = L.LlamaDecoder(w, "macko")
dec.reset()
for _ in range(4):
    dec.step()
torch.cuda.synchronize()
bad += int(not torch.isfinite(dec.logits.float()).all())
print("mismatches", bad)
