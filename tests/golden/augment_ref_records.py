"""Add pattern digests and value moments (tests/_digest.hierarchy_record) to a
reference record made before those fields existed, from the hierarchy npz
make_golden_large.py --save wrote.  Used once per record:

    python tests/golden/augment_ref_records.py c3 /tmp/refh/c3_ref_hierarchy.npz
"""
import json
import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from _digest import hierarchy_record  # noqa: E402

cfg, npz = sys.argv[1], sys.argv[2]
z = np.load(npz)
L = int(z["nlev"])
get = lambda p: sp.csr_matrix((z[p + "_data"], z[p + "_indices"], z[p + "_indptr"]),  # noqa: E731
                              shape=tuple(z[p + "_shape"]))
mats = [get(f"A{k}") for k in range(L)]
pros = [get(f"P{k}") for k in range(L - 1)]
path = os.path.join(HERE, f"{cfg}_ref.json")
rec = json.load(open(path))
new = hierarchy_record(mats, pros)
assert new["A_sha256"] == rec["A_sha256"] and new["P_sha256"] == rec["P_sha256"], "npz is not this record's hierarchy"
rec.update(new)
json.dump(rec, open(path, "w"), indent=1)
print(cfg, "augmented")
