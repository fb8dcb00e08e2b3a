"""Shared-memory bank conflicts of the byte-step table probes (simulation).

For real encoded streams (alpha 1.8, gamma 0.05, T 256), the (state, byte)
index every lane of a warp probes at each byte step, and the wavefronts a
probe costs under several table layouts (max distinct rows per bank).
python tools/bank_sim.py   (CPU; result in profiles/r2_bank_sim.txt)
"""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from paper_2510_02676_b200 import codec
x = codec.synth(1.8, 0.05, 4096*4096, 1)
t = codec.encode_tensor(x, 256)
fsm, cm, ok = codec.fsm_tables(t.lengths)
enc = np.asarray(t.encoded); n_win = (enc.size-2)//8
padded = np.concatenate([enc, np.zeros(128, np.uint8)])
g = np.asarray(t.gaps)
gaps = np.stack([g >> 4, g & 15], 1).reshape(-1)[:n_win]
# per lane (8 windows): bytes from gap0
ntiles = 200
bits_all = np.unpackbits(padded)
res = {}
layouts = {
 'cur byte&31': lambda s,b: b & 31,
 'stride257 (b+s)': lambda s,b: (b + s) & 31,
 'b^(s*7)': lambda s,b: (b ^ (s*7)) & 31,
 'b^(b>>5)*9': lambda s,b: (b ^ ((b >> 5)*9)) & 31,
 'b^s^(b>>5)*9': lambda s,b: (b ^ s ^ ((b >> 5)*9)) & 31,
 'random hash': lambda s,b: ((s*256+b)*2654435761 >> 11) & 31,
}
tot = {k:0 for k in layouts}; steps=0
for tile in range(ntiles):
    states = np.zeros((32, 66), np.int64); bytes_ = np.zeros((32,66), np.int64)
    for lane in range(32):
        w0 = tile*256 + lane*8
        g0 = int(gaps[w0])
        b = bits_all[64*w0 + g0: 64*w0 + g0 + 66*8]
        by = np.packbits(b)
        st = 0
        for j in range(66):
            states[lane, j] = st; bytes_[lane, j] = by[j]
            st = (int(fsm[st, by[j]]) >> 8) & 0xFF
    for j in range(66):
        for k, f in layouts.items():
            bk = f(states[:, j], bytes_[:, j])
            addr = states[:, j]*256 + bytes_[:, j]
            # wavefronts = max over banks of distinct addresses
            wf = 0
            for bank in range(32):
                m = bk == bank
                if m.any(): wf = max(wf, len(np.unique(addr[m])))
            tot[k] += wf
        steps += 1
for k in layouts: print(f"{k:20s} {tot[k]/steps:.2f} wavefronts/LDS")
# state distribution
print("state hist", np.bincount(states.reshape(-1), minlength=16))
