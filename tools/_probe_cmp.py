import sys
import numpy as np
a, b = np.load("/tmp/ftop_0.npy"), np.load("/tmp/ftop_1.npy")
sa, sb = np.load("/tmp/st_0.npy"), np.load("/tmp/st_1.npy")
d = np.where(~((a == b) | (np.isnan(a) & np.isnan(b))).all(axis=1))[0]
print("ftop differs for", len(d), "of", len(a), "candidates; first", d[:10])
print("states differ for", int((sa != sb).sum()))
for i in d[:3]:
    j = np.where(a[i] != b[i])[0]
    print(i, j[:5], a[i, j[:5]], b[i, j[:5]])
