import sys, numpy as np
sys.path.insert(0, ".")
from paper_1103_3105_b200 import Database
rng = np.random.default_rng(1)
n = 200000
b = rng.integers(0, 2000, n); t = b * 10 + rng.integers(0, 10, n); a = b * 1000 + rng.integers(0, 1000, n)
pw = np.stack([a, t, b, rng.integers(0, 1000, n)], 1).astype(np.uint32).reshape(-1)
class B: pass
bk = B(); bk.type = np.zeros(n, np.uint8); bk.param_off = (np.arange(n + 1) * 4).astype(np.uint32); bk.param_words = pw
img = {"br_bal": np.zeros(2000, np.int64), "tel_bal": np.zeros(20000, np.int64), "acc_bal": np.zeros(2000000, np.int64)}
db = Database(1, (2000, 10, 1000, 0), n, img)
db.trace_rounds(True)
for it in range(3):
    db.submit(bk); s = db.execute("kset")
tr = db.round_ns(s["ksets"]).astype(np.int64)
print(f"python TPC-B: ksets {s['ksets']} exec_ms {s['ms_exec']:.3f} mean round {np.diff(tr[:, 0]).mean() / 1e3:.2f} us")
