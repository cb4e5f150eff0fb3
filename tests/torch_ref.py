"""Plain PyTorch fp32 restatement of the reference forward (model.cpp:149-220)
and score head (model.cpp:294-352). Test-only numerics reference for the
floating-point kernels; parity proper is against the CPU oracle (oracle/).
"""
import math

import numpy as np


def _bf16(x):
    import torch
    return x.bfloat16().float()


def forward_items(w, cfg, prefix, items, device, round_weights=True, soft_rows=None):
    """Scores of each item (dict task -> prob) via independent naive prefill."""
    import torch
    t = {k: torch.as_tensor(v) for k, v in w.tensors().items()}
    d, H, F, L, V = cfg.d_model, cfg.n_heads, cfg.d_ff, cfg.n_layers, cfg.vocab_size
    hd = d // H
    rw = _bf16 if round_weights else (lambda z: z)
    dev = lambda z: z.to(device)
    tok = dev(t["tok_emb"].view(V, d))
    pos = dev(t["pos_emb"].view(cfg.max_seq, d))
    layers = []
    for l in range(L):
        p = f"layers.{l}."
        layers.append(dict(
            wq=dev(rw(t[p + "wq"].view(d, d))), wk=dev(rw(t[p + "wk"].view(d, d))),
            wv=dev(rw(t[p + "wv"].view(d, d))), wo=dev(rw(t[p + "wo"].view(d, d))),
            ln1=dev(t[p + "ln1_gain"]), ln2=dev(t[p + "ln2_gain"]),
            win=dev(rw(t[p + "w_mlp_in"].view(d, F))), wout=dev(rw(t[p + "w_mlp_out"].view(F, d)))))
    lnf = dev(t["ln_f_gain"])
    wv = dev(t["w_vocab"].view(d, V))

    def ln(x, g):
        m = x.mean(-1, keepdim=True)
        v = ((x - m) ** 2).mean(-1, keepdim=True)
        return (x - m) / torch.sqrt(v + 1e-5) * g

    out = []
    for i, it in enumerate(items):
        T = len(prefix) + (len(it) if soft_rows is None else soft_rows[i].shape[0])
        if soft_rows is None:
            ids = torch.as_tensor(list(prefix) + list(it), device=device)
            x = tok[ids] + pos[:T]
        else:
            ids = torch.as_tensor(list(prefix), device=device, dtype=torch.long)
            rows = torch.cat([tok[ids], torch.as_tensor(soft_rows[i], device=device)], 0)
            x = rows + pos[:T]
        mask = torch.ones(T, T, dtype=torch.bool, device=device).tril()
        for lw in layers:
            h = ln(x, lw["ln1"])
            q = (h @ lw["wq"]).view(T, H, hd)
            k = (h @ lw["wk"]).view(T, H, hd)
            v = (h @ lw["wv"]).view(T, H, hd)
            s = torch.einsum("qhd,khd->hqk", q, k) / math.sqrt(hd)
            s = s.masked_fill(~mask[None], float("-inf"))
            a = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v).reshape(T, d)
            x = x + a @ lw["wo"]
            h = ln(x, lw["ln2"])
            x = x + torch.nn.functional.gelu(h @ lw["win"]) @ lw["wout"]
        hl = ln(x[-1], lnf)
        lg = hl @ wv
        diff = float(lg[cfg.no_token_id]) - float(lg[cfg.yes_token_id])
        rel = math.exp(-diff) / (1 + math.exp(-diff)) if diff > 0 else 1 / (1 + math.exp(diff))
        tasks = {"relevance": rel}
        for hs in cfg.head_specs:
            hw = dev(t[f"heads.{hs.name}.w"].view(d, hs.arity))
            hb = dev(t[f"heads.{hs.name}.b"])
            z = (hl @ hw + hb).double().cpu().numpy()
            if hs.arity == 1:
                tasks[hs.name] = float(1 / (1 + np.exp(-z[0])))
            else:
                e = np.exp(z - z.max())
                tasks[hs.name] = float(e[0] / e.sum())
        out.append(tasks)
    return out
