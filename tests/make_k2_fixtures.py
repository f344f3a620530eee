"""Writes tests/golden/k2_fixtures.json: the reference replay's reported triples
and per-line first-detection keys for the trace cases of tests/test_oracle.py
(run here, where oracle/_ref is built from /root/reference)."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_bind as ob  # noqa: E402
from test_oracle import _cases  # noqa: E402

out = {}
for name, ev, bs, shm in _cases():
    rc, tri, n, lf = ob.ref_detect(ob.make_trace(ev, bs, shm))
    assert rc == 0
    out[name] = {"n": int(n), "triples": [list(map(int, t)) for t in ob.sorted_triples(tri).tolist()],
                 "line_first": {str(l): int(lf[l]) for l in np.nonzero(lf != ob.TS_NONE)[0]}}
json.dump(out, open(os.path.join(HERE, "golden", "k2_fixtures.json"), "w"), separators=(",", ":"))
print("wrote", len(out))
