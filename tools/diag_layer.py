"""GPU diagnostic: replay one layer with the kernel entry points, check each step."""
import sys, os, math, ctypes as C, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_07309_b200 as sr
from paper_2602_07309_b200._capi import lib
dev = torch.device('cuda:0')
vp = lambda t: C.c_void_p(t.data_ptr())
def ok(s): assert s == 0, lib.sr_last_error().decode()
for (d, H, F) in [(256, 2, 256), (128, 1, 128), (512, 8, 512)]:
    cfg = sr.ModelConfig(n_layers=1, d_model=d, n_heads=H, d_ff=F, head_specs=sr.ModelConfig.default_toy().head_specs)
    w = sr.init_model(cfg, 2026, "fan_in"); t = {k: torch.as_tensor(v).to(dev) for k, v in w.tensors().items()}
    hd = d // H; tq = 64; lens = [32, 32]; M = tq + sum(lens)
    rng = np.random.default_rng(7)
    toks = torch.as_tensor(rng.integers(0, 256, M), device=dev)
    pos = torch.as_tensor(list(range(tq)) + [tq + j for L in lens for j in range(L)], device=dev)
    x = t['tok_emb'].view(-1, d)[toks] + t['pos_emb'].view(-1, d)[pos]
    spans = [[0, 0, 0, 0]] * tq; cur = tq
    for L in lens:
        spans += [[0, tq, cur, 0]] * L; cur += L
    spn = np.asarray(spans, np.int32).reshape(-1)
    p = 'layers.0.'
    WT = lambda n, K, N: t[p + n].view(K, N).T.contiguous().bfloat16()
    wqkv = torch.cat([WT('wq', d, d), WT('wk', d, d), WT('wv', d, d)], 0).contiguous()
    def lnref(x, g):
        m = x.mean(-1, keepdim=True); v = ((x - m) ** 2).mean(-1, keepdim=True); return (x - m) / torch.sqrt(v + 1e-5) * g
    xn = torch.zeros(M, d, dtype=torch.bfloat16, device=dev)
    ok(lib.sr_kernel_layernorm(vp(x), vp(t[p + 'ln1_gain']), vp(xn), M, d, None))
    print(d, H, "ln1 dev", (xn.float() - lnref(x, t[p + 'ln1_gain'])).abs().max().item())
    qkv = torch.zeros(M, 3 * d, dtype=torch.bfloat16, device=dev)
    ok(lib.sr_kernel_gemm(vp(xn), vp(wqkv), M, 3 * d, d, vp(qkv), 3 * d, 0, None))
    print(d, H, "qkv dev", (qkv.float() - xn.float() @ wqkv.float().T).abs().max().item())
    att = torch.zeros(M, d, dtype=torch.bfloat16, device=dev)
    ok(lib.sr_kernel_attention(vp(qkv), spn.ctypes.data_as(C.POINTER(C.c_int32)), M, H, hd, vp(att), None))
    q = qkv[:, :d].float().view(M, H, hd); k = qkv[:, d:2*d].float().view(M, H, hd); v = qkv[:, 2*d:].float().view(M, H, hd)
    sp = torch.as_tensor(spans, device=dev); keys = torch.arange(M, device=dev); rows = keys[:, None]
    allowed = ((keys[None] >= sp[:, 0:1]) & (keys[None] < sp[:, 1:2])) | ((keys[None] >= sp[:, 2:3]) & (keys[None] <= rows))
    s = torch.einsum('qhd,khd->hqk', q, k) / math.sqrt(hd); s = s.masked_fill(~allowed[None], float('-inf'))
    aref = torch.einsum('hqk,khd->qhd', torch.softmax(s, -1), v).reshape(M, d)
    e = (att.float() - aref).abs()
    print(d, H, "attn dev", e.max().item(), "per-head max", [round(e[:, h*hd:(h+1)*hd].max().item(), 4) for h in range(H)], "|a|", aref.abs().max().item())
    x2 = x.clone()
    wo = WT('wo', d, d)
    ok(lib.sr_kernel_gemm(vp(att), vp(wo), M, d, d, vp(x2), d, 2, None))
    print(d, H, "o-resid dev", (x2 - (x + att.float() @ wo.float().T)).abs().max().item())
