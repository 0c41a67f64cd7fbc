"""Deep-learning (DL) oracle, serial fp64 (TEST INFRASTRUCTURE ONLY).

PAPER.md §V-B: "a convolutional neural network that projects 2
input images to low dimensional embeddings and combines the embeddings using
a dense layer".  Node names from Fig. 6 (L702-710): CONV x4, POOL x2,
CONCAT, DOT.  Architecture is a SURVEY §8(c2) DL reading (DESIGN.md R-DL),
shared ("siamese") weights for both branches:

    c1 = ReLU(conv3x3, stride 2, pad 1 (x; W1 in 8x3x3x1))   NHWC, cross-correlation
    p  = meanpool 2x2 stride 2 (c1)                           (odd trailing row/col dropped)
    c2 = ReLU(conv3x3, stride 2, pad 1 (p; W2 in 16x3x3x8))
    z  = [vec(c2_x); vec(c2_y)]     (row-major NHWC flatten)
    r  = sum_i z_i wd_i

Pins (tests/test_oracle_dl.py): conv equals torch.nn.functional.conv2d in
float64 on the CPU (stride 2, padding 1) followed by ReLU; delta kernel ->
strided copy; pooling a constant -> the constant; dot within 1e-12 of
math.fsum; brute force on 9x9 inputs.
"""
import numpy as np


def conv3x3s2(x, w):
    """out[p,q,k] = ReLU(sum_{a,b,c} w[k,a,b,c] x[2p+a-1, 2q+b-1, c]), zero pad.

    x: (H, W, Cin) ; w: (Cout, 3, 3, Cin) ; out: (ceil(H/2), ceil(W/2), Cout).
    """
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 2:
        x = x[:, :, None]
    w = np.asarray(w, dtype=np.float64)
    h, wd, cin = x.shape
    cout = w.shape[0]
    ho, wo = (h + 1) // 2, (wd + 1) // 2
    pad = np.zeros((h + 2 + 1, wd + 2 + 1, cin))
    pad[1:1 + h, 1:1 + wd] = x
    out = np.zeros((ho, wo, cout))
    for a in range(3):
        for b in range(3):
            patch = pad[a:a + 2 * ho:2, b:b + 2 * wo:2, :]  # x[2p+a-1, 2q+b-1, :]
            out += np.einsum("pqc,kc->pqk", patch, w[:, a, b, :])
    return np.maximum(out, 0.0)


def pool2x2(x):
    """Mean of each 2x2 window, stride 2; trailing odd row/column dropped."""
    x = np.asarray(x, dtype=np.float64)
    h, w = x.shape[0] // 2, x.shape[1] // 2
    x = x[:2 * h, :2 * w]
    return 0.25 * (x[0::2, 0::2] + x[0::2, 1::2] + x[1::2, 0::2] + x[1::2, 1::2])


def concat(a, b):
    return np.concatenate([np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()])


def dot(z, wd):
    return float(np.dot(np.asarray(z, np.float64), np.asarray(wd, np.float64)))


def dl(x, y, w1, w2, wd):
    """The DL DAG in program order."""
    w1 = np.asarray(w1, np.float64).reshape(8, 3, 3, 1)
    w2 = np.asarray(w2, np.float64).reshape(16, 3, 3, 8)
    c1x = conv3x3s2(x, w1)
    c1y = conv3x3s2(y, w1)
    px = pool2x2(c1x)
    py = pool2x2(c1y)
    c2x = conv3x3s2(px, w2)
    c2y = conv3x3s2(py, w2)
    z = concat(c2x, c2y)
    r = dot(z, wd)
    return dict(c1x=c1x, c1y=c1y, px=px, py=py, c2x=c2x, c2y=c2y, z=z, r=r)
