"""Prototype: the fast-mode NDFT as a sign-split bf16 GEMM through cuBLAS (torch.mm).

Measures what a tensor-core formulation could reach at C2 and its accuracy against
the fp64 oracle restatement, before writing the tcgen05 kernel (tools/, not product).
  Re X = S_r Wr + X_r sgn(Wr) - S_i Wi - X_i sgn(Wi)
  Im X = S_r Wi + X_r sgn(Wi) + S_i Wr + X_i sgn(Wr)
"""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1402_0532_b200 import ndft_batch
from paper_1402_0532_b200.twiddle import twiddle_table

N, B = 1024, 65536
dev = 'cuda'
def split2(t):
    hi = t.to(torch.bfloat16); lo = (t - hi.float()).to(torch.bfloat16); return hi, lo
tw = torch.from_numpy(np.asarray(twiddle_table(N).entries)).to(dev)
idx = (torch.arange(N, device=dev)[:, None] * torch.arange(N, device=dev)[None, :]) % N
W = tw[idx].to(torch.complex64)  # [k, n]
Wr, Wi = W.real, W.imag
# B operand rows o = 2k + c_out, cols K = 2n + c_in
def inter(a, b, c, d):  # rows 2k: [a(n,re) b(n,im)], rows 2k+1: [c, d]
    o = torch.empty(2 * N, 2 * N, device=dev)
    o[0::2, 0::2] = a; o[0::2, 1::2] = b; o[1::2, 0::2] = c; o[1::2, 1::2] = d
    return o
Wv = inter(Wr, -Wi, Wi, Wr)
Ws = inter(torch.sign(Wr), -torch.sign(Wi), torch.sign(Wi), torch.sign(Wr))
W0, W1 = split2(Wv); Ws16 = Ws.to(torch.bfloat16)
Bcat = torch.cat([W0, W1, Ws16, Ws16], 1).contiguous()  # [2N, 8N]
g = torch.Generator(device=dev).manual_seed(5)
x = torch.complex(torch.randn(B, N, device=dev, generator=g), torch.randn(B, N, device=dev, generator=g)) / 2 ** 0.5
xv = torch.view_as_real(x).reshape(B, 2 * N)
def prep(xv):
    S = torch.sign(xv).to(torch.bfloat16); X0, X1 = split2(xv)
    return torch.cat([S, S, X0, X1], 1)
def run():
    A = prep(xv)
    return torch.mm(A, Bcat.t(), out_dtype=torch.float32)
for _ in range(3): D = run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
A = prep(xv)
e0.record(); 
for _ in range(5): D = torch.mm(A, Bcat.t(), out_dtype=torch.float32)
e1.record(); torch.cuda.synchronize(); t_mm = e0.elapsed_time(e1) / 5
e0.record();
for _ in range(5): D = run()
e1.record(); torch.cuda.synchronize(); t_all = e0.elapsed_time(e1) / 5
flop = 2.0 * B * 2 * N * 8 * N
print(f"mm {t_mm:.3f} ms = {flop / t_mm / 1e9:.0f} TFLOP/s ; prep+mm {t_all:.3f} ms")
y = torch.view_as_complex(D.view(B, N, 2))
yf = ndft_batch(x, mode='fast')
rows = torch.arange(0, B, 997, device=dev)
xs = x[rows].cpu().numpy().astype(np.complex128)
twn = np.asarray(twiddle_table(N).entries).astype(np.complex64).astype(np.complex128)
Wn = twn[(np.arange(N)[:, None] * np.arange(N)[None, :]) % N]
sg = np.sign
ref = (sg(xs.real) @ Wn.real.T + xs.real @ sg(Wn.real).T - sg(xs.imag) @ Wn.imag.T - xs.imag @ sg(Wn.imag).T) + 1j * (
    sg(xs.real) @ Wn.imag.T + xs.real @ sg(Wn.imag).T + sg(xs.imag) @ Wn.real.T + xs.imag @ sg(Wn.real).T)
l1 = np.abs(ref).sum(1)
for name, yy in (('tc', y), ('fast', yf)):
    d = np.abs(yy[rows].cpu().numpy() - ref)
    print(name, 'max|d|/l1', (d.max(1) / l1).max(), 'l1d/l1', (d.sum(1) / l1).max())
