"""Phase offset between the two streams of one SM in the dense forward (diagnostics)."""
import os
import runpy
import sys

import numpy as np

sys.argv = [sys.argv[0], "dense"]
g = runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "timing.py"), run_name="x")
d = g["bufs"]["scfa_attn_fwd"].view(g["grid"], g["TILES"], 16).cpu().numpy().astype(np.float64)
for cta in (0, 10, 70):
    a, b = d[2 * cta], d[2 * cta + 1]
    na, nb = int((a[:, 0] > 0).sum()), int((b[:, 0] > 0).sum())
    sa, sb = a[:na, 1], b[:nb, 1]
    per = np.median(np.diff(sa))
    offs = []
    for t in sa[5:na - 5]:
        j = np.searchsorted(sb, t)
        if 0 < j < nb:
            offs.append(min(t - sb[j - 1], sb[j] - t) / per)
    h = np.histogram(offs, bins=5, range=(0, 0.5))[0]
    print(f"sm {cta}: period {per:.0f}  offset/period histogram [0,.1,.2,.3,.4,.5]: {h.tolist()}  rows median a {np.median(a[:na,2]-a[:na,1]):.0f}")
