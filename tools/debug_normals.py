import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2002_01119_b200 import objectives
for ent, n in [((2**40, 6), 5_000_000), ((3, 0, 5, 1), 20_000_000), ((11,), 20_000_000)]:
    got = objectives.standard_normal(n, *ent).cpu().numpy()
    ref = np.random.default_rng(np.random.SeedSequence(ent)).standard_normal(n)
    bad = np.nonzero(got != ref)[0]
    tail = np.abs(ref) > 3.6541528853610088
    ulps = np.abs(got.view(np.int64) - ref.view(np.int64))
    print(json.dumps({"ent": [str(e) for e in ent], "n": n, "mismatch": int(len(bad)),
                      "first": [int(x) for x in bad[:10]],
                      "tail_frac_of_bad": float(tail[bad].mean()) if len(bad) else None,
                      "tail_total": int(tail.sum()),
                      "max_ulps": int(ulps[bad].max()) if len(bad) else 0,
                      "contiguous_run": bool(len(bad) > 1 and np.all(np.diff(bad[:50]) == 1))}), flush=True)
