"""Per-CTA analysis of a VXB_PROF_DUMP file of tile_kernel (8 timestamps per
(phase, CTA): U end, B end, C end, N end, phase start, B pass 1 / reservation
/ pass 2 ends)."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
G = int(sys.argv[2]) if len(sys.argv) > 2 else 148
K = 8
P = a.size // (G * K)
a = a.reshape(P, G, K)
st = a[:, :, 4]
rel = (a[:, :, [0, 1, 2, 3, 5, 6, 7]] - st[:, :, None]) / 1e3
ph = slice(5, P - 2)
print("phases", P)
m = np.where(rel[ph] > -1e6, rel[ph], np.nan)
print("mean end rel to CTA start: U %.1f B %.1f C %.1f N %.1f | B pass1 %.1f reserve %.1f pass2 %.1f" % tuple(np.nanmean(m, axis=(0, 1))))
dur = (st[1:] - st[:-1]) / 1e3
print("phase duration mean %.1f us" % dur[ph].mean())
spread = (st.max(1) - st.min(1)) / 1e3
print("start spread per phase: mean %.1f max %.1f" % (spread[ph].mean(), spread[ph].max()))
late = ((st - st.mean(1, keepdims=True)) / 1e3)[ph].mean(0)
print("latest CTAs", np.argsort(-late)[:8], np.round(np.sort(-late)[:8] * -1, 1))
print("earliest CTAs", np.argsort(late)[:8], np.round(np.sort(late)[:8], 1))
Bend = a[:, :, 1]
wait = (Bend[:-1].max(1)[:, None] - st[1:]) / 1e3
print("next-phase consumer wait: mean %.1f us, CTAs waiting %.0f%%" % (np.clip(wait[ph], 0, None).mean(), 100 * (wait[ph] > 0).mean()))
print("B duration mean %.1f" % (rel[ph, :, 1] - rel[ph, :, 0]).mean())
