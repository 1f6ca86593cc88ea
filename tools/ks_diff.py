import sys, numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
print("its equal", np.array_equal(a["its"], b["its"]), "max |dits|", np.abs(a["its"] - b["its"]).max(),
      "status equal", np.array_equal(a["status"], b["status"]))
for k in ("dx", "dy", "ds", "dyd"):
    x, y = a[k], b[k]
    num = np.linalg.norm(x - y, axis=1); den = np.linalg.norm(y, axis=1)
    print(k, "max rel", (num / np.maximum(den, 1e-300)).max())
