import sys, numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    x, y = a[k], b[k]
    same = x.shape == y.shape and np.array_equal(x, y)
    print(k, x.shape, y.shape, "bitwise" if same else ("maxdiff %.3g" % np.max(np.abs(x - y)) if x.shape == y.shape else "SHAPE"))
