"""Compare the step's exact partial sums (accum) of fast vs vec kernels."""
import os, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from tests.golden_util import load_case, config_for
from paper_1705_09339_b200.training import train_engine

rec, ov = load_case(sys.argv[1] if len(sys.argv) > 1 else "c3small")
cfg = config_for(ov)
fr = rec["frames"]; n = int(rec["n_train"])
out = {}
for kern in ("fast", "vec"):
    os.environ["COG_KERNEL"] = kern
    e = train_engine(fr[:n], cfg)
    got = []
    e.reducer = lambda acc: got.append(acc.clone().cpu().numpy().astype(np.uint64))
    for t in range(3):
        e.process_frame(fr[n + t]).__class__
    out[kern] = got
    print(kern, "G", e.dev.n_groups, "words", e.dev.words)
for t in range(3):
    a, b = out["fast"][t][0], out["vec"][t][0]
    d = np.nonzero(a != b)[0]
    print("frame", t, "differing words", d.tolist()[:20])
    for i in d[:12]:
        print("   ", i, int(a[i]), int(b[i]))

# expected partial words from the exported kinds / confidences / frame
for kern in ("fast", "vec"):
    os.environ["COG_KERNEL"] = kern
    e = train_engine(fr[:n], cfg)
    got = []
    e.reducer = lambda acc: got.append(acc.clone().cpu().numpy().astype(np.uint64))
    for t in range(3):
        e.process_frame(fr[n + t])
        kinds, conf = e.last_kinds, e.last_confidence
        gid = e.group_id
        d = e.depth
        for c in range(d):
            sel = (kinds[c] == 1) & (gid == 0)
            tot = np.floor(conf[c][sel] * 2.0 ** 52).sum() / 2.0 ** 52
            w = got[t][0]
            base = 7 * d + 1 + c * e.dev.n_groups * 6
            acc = float(w[base + 2]) * 2.0 ** -26 + float(w[base + 3]) * 2.0 ** -52
            print(kern, t, "plane", c, "hits", int(sel.sum()), int(w[base]), "conf sum", tot, "accum", acc, "sv", int(fr[n + t][c].ravel()[sel].astype(np.int64).sum()), int(w[base + 1]))
