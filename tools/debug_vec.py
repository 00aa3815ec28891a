"""Compare COG_KERNEL=vec against the scalar fast kernel frame by frame."""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from tests.golden_util import load_case, config_for
from paper_1705_09339_b200.training import train_engine

name = sys.argv[1] if len(sys.argv) > 1 else "c3small"
rec, ov = load_case(name)
cfg = config_for(ov)
fr = rec["frames"]; n = int(rec["n_train"])
engs = {}
for kern in ("fast", "vec"):
    os.environ["COG_KERNEL"] = kern
    e = train_engine(fr[:n], cfg)
    engs[kern] = e
a, b = engs["fast"], engs["vec"]
for t in range(fr.shape[0] - n):
    os.environ["COG_KERNEL"] = "fast"; ma, sa = a.process_frame(fr[n + t])
    os.environ["COG_KERNEL"] = "vec"; mb, sb = b.process_frame(fr[n + t])
    bad = []
    ga, gb = a.group_mu, b.group_mu
    print(t, "gmu fast", ga.ravel()[:4], "vec", gb.ravel()[:4], "gvar", a.group_var.ravel()[:2], b.group_var.ravel()[:2])
    ca, cb = a.last_confidence, b.last_confidence
    if not np.allclose(ca, cb, atol=1e-6):
        d = np.argwhere(~np.isclose(ca, cb, atol=1e-6))[:4]
        bad.append(f"conf at {d.tolist()} fast {[ca[tuple(q)] for q in d]} vec {[cb[tuple(q)] for q in d]} kinds {[a.last_kinds[tuple(q)] for q in d]} {[b.last_kinds[tuple(q)] for q in d]}")
    if not np.array_equal(ma.labels, mb.labels): bad.append("mask")
    if sa.as_row() != sb.as_row(): bad.append(f"stats {sa.as_row()} {sb.as_row()}")
    if not np.array_equal(a.last_kinds, b.last_kinds):
        d = np.argwhere(a.last_kinds != b.last_kinds)[:5]
        bad.append(f"kinds at {d.tolist()} fast {[a.last_kinds[tuple(x)] for x in d]} vec {[b.last_kinds[tuple(x)] for x in d]}")
    for nm in ("mu", "var", "w", "count", "mode_ref", "chp_prev", "last_label", "streak", "hits", "clock", "waking", "last_active"):
        x, y = getattr(a, nm), getattr(b, nm)
        if not np.array_equal(x, y):
            d = np.argwhere(x != y)[:3]
            bad.append(f"{nm} at {d.tolist()} fast {[x[tuple(q)] for q in d]} vec {[y[tuple(q)] for q in d]}")
    if bad:
        print("frame", t, *bad, sep="\n  ")
        break
else:
    print("identical over", fr.shape[0] - n, "frames")
