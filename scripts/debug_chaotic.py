import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, golden_cases as G
from oracle import cgh_oracle as O
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.runtime import precision
MAN = G.manifest()["cases"]
for name in sorted(MAN):
    if "chaotic" not in str(MAN[name].get("tags", "")) and name not in ("gs_backprop_fresnel_32_pl16",): continue
    rec = MAN[name]; cfg, target, illum = G.build(rec); arrs = G.load_arrays(name)
    cfg.iterations = 1
    _, ref = O.gs(cfg, target, illum, keep_fields=(1,))
    with precision("fp32"):
        _, fld, rep, trace = A.gs_field(cfg, target, illum)
    e = np.linalg.norm(fld - ref.fields[1]) / np.linalg.norm(ref.fields[1])
    d = np.abs(fld - ref.fields[1]); i = np.unravel_index(np.argmax(d), d.shape)
    print(name, "field", e, "trace", abs(trace[0][1] - arrs["trace"][0]) / arrs["trace"][0], "worst px", i, d[i], abs(ref.fields[1][i]))
