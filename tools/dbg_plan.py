import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2105_11815_b200 as skh
from synth import configs, device
cfg = configs.ALL[sys.argv[1] if len(sys.argv) > 1 else 'C2']
At = device.dense_colmajor(cfg); b = device.rhs(cfg)
op = skh.RhtDenseColMajor(cfg.n, cfg.m, cfg.s, cfg.d)
op(cfg.seed, At, b); torch.cuda.synchronize()
n_pad = 1 << (cfg.n - 1).bit_length()
ntiles = n_pad // 4096
al = lambda x: (x + 255) // 256 * 256
jcap = 24 * cfg.s + 16
words = al(4 * ntiles * jcap * 256)
tot = op.ws.numel()
lists = tot - words - al(4 * ntiles)
ws = op.ws
hdr = ws[lists + words: lists + words + 4 * ntiles].view(torch.int32).cpu().numpy()
print(cfg.name, 'ws', tot, 'hdr', np.unique(hdr, return_counts=True))
w = ws[lists: lists + words].view(torch.int32).cpu().numpy().view(np.uint32)
t0 = w[: jcap * 256].reshape(jcap // 4, 256, 4).transpose(1, 0, 2).reshape(256, jcap)
print('tile0 valid per thread', ((t0 >> 29) & 1).sum(1)[:40])
# bank multiplicity per (half-warp, step) on tile 0: the consumer's tile reads
J = int(hdr[0])
t0 = t0[:, :J]
tot = ideal = 0
for u in range(16):
    c = [32 * (u >> 1) + 16 * (u & 1) + cl for cl in range(16)]
    for j in range(J):
        ws_ = t0[c, j]
        act = ws_[(ws_ & ((1 << 28) | (1 << 30) | 0xFFFFFFF)) != 0]
        pads = len(ws_) - len(act)
        banks = np.bincount((act & 4095) & 15, minlength=16)
        if pads: banks[0] += 1
        tot += banks.max(); ideal += 1
print('J', J, 'mean wavefronts per half-warp step', tot / ideal)
