"""Image-processing (IMG) oracle, serial fp64 (TEST INFRASTRUCTURE ONLY).

PAPER.md §V-B: "an image processing pipeline that combines a
sharpened picture with copies blurred at low and medium frequencies [29], to
sharpen the edges, soften everything else, and enhance the subject."  Node
names from Fig. 6 (L759-769): BLUR x3, SOBEL x2, MAX, MIN, EXTEND, UNSHARPEN,
COMBINE x2.  The exact pipeline, constants and zero padding are SURVEY
§8(c2) IMG readings (DESIGN.md R-IMG); the paper prints no formulas.

    bs = blur(img, d=3, s2=0.1)    bl = blur(img, d=5, s2=10)   bu = blur(img, d=3, s2=5)
    ms = sobel(bs)                 ml = sobel(bl)
    mx = max(ml)                   mn = min(ml)
    ml = min(1, 5 (ml - mn)/(mx - mn))                           (in place)
    iu = clamp(img (1+a) - bu a, 0, 1),  a = 0.5
    i2 = iu ml + bl (1 - ml)
    i3 = i2 ms + bs (1 - ms)

Pins (tests/test_oracle_img.py): blur and sobel equal scipy.ndimage.correlate
/ scipy.ndimage.sobel with zero padding; Gaussian taps have the closed-form
ratios exp(-1/(2 s2)) and sum to 1; constant image -> blur constant, sobel 0
in the interior; unit ramp -> |grad| = 8; combine with m=1 / m=0; brute force
on 7x9 images.
"""
import numpy as np

BLUR_S = (3, 0.1)    # (diameter, sigma^2) -- readings, parity unpinned (constant)
BLUR_L = (5, 10.0)
BLUR_U = (3, 5.0)
UNSHARP_AMOUNT = 0.5
EXTEND_FACTOR = 5.0

SOBEL_X = np.array([[-1.0, 0.0, 1.0], [-2.0, 0.0, 2.0], [-1.0, 0.0, 1.0]])
SOBEL_Y = SOBEL_X.T


def gaussian(diameter, sigma2):
    """G[a,b] ~ exp(-(a^2+b^2)/(2 sigma^2)), a,b in [-r, r], normalised to sum 1."""
    r = diameter // 2
    a = np.arange(-r, r + 1, dtype=np.float64)
    g = np.exp(-(a[:, None] ** 2 + a[None, :] ** 2) / (2.0 * sigma2))
    return g / g.sum()


def correlate_zero(img, taps):
    """out[i,j] = sum_{a,b} taps[a,b] img[i+a-r, j+b-r], out-of-range taps read 0."""
    img = np.asarray(img, dtype=np.float64)
    h, w = img.shape
    r = taps.shape[0] // 2
    pad = np.zeros((h + 2 * r, w + 2 * r))
    pad[r:r + h, r:r + w] = img
    out = np.zeros((h, w))
    for a in range(taps.shape[0]):
        for b in range(taps.shape[1]):
            out += taps[a, b] * pad[a:a + h, b:b + w]
    return out


def blur(img, diameter, sigma2):
    """BLUR (Fig. 6): 2-D Gaussian, zero padding."""
    return correlate_zero(img, gaussian(diameter, sigma2))


def sobel(img):
    """SOBEL (Fig. 6): |grad| = sqrt(gx^2 + gy^2), 3x3 Sobel taps."""
    gx = correlate_zero(img, SOBEL_X)
    gy = correlate_zero(img, SOBEL_Y)
    return np.sqrt(gx * gx + gy * gy)


def maximum(m):
    return float(np.max(m))


def minimum(m):
    return float(np.min(m))


def extend(m, mx, mn, factor=EXTEND_FACTOR):
    """EXTEND (Fig. 6): m = min(1, factor (m - mn)/(mx - mn)); if mx == mn, m = 0."""
    m = np.asarray(m, dtype=np.float64)
    if mx == mn:
        return np.zeros_like(m)
    return np.minimum(1.0, factor * (m - mn) / (mx - mn))


def unsharpen(img, blurred, amount=UNSHARP_AMOUNT):
    """UNSHARPEN (Fig. 6): clamp(x (1+a) - blur a, 0, 1)."""
    x = np.asarray(img, dtype=np.float64)
    return np.clip(x * (1.0 + amount) - np.asarray(blurred, np.float64) * amount, 0.0, 1.0)


def combine(x, y, m):
    """COMBINE (Fig. 6): x m + y (1 - m)."""
    x, y, m = (np.asarray(v, dtype=np.float64) for v in (x, y, m))
    return x * m + y * (1.0 - m)


def img_pipeline(img):
    """The IMG DAG in program order; returns every intermediate."""
    img = np.asarray(img, dtype=np.float64)
    bs = blur(img, *BLUR_S)
    bl = blur(img, *BLUR_L)
    bu = blur(img, *BLUR_U)
    ms = sobel(bs)
    ml0 = sobel(bl)
    mx = maximum(ml0)
    mn = minimum(ml0)
    ml = extend(ml0, mx, mn)
    iu = unsharpen(img, bu)
    i2 = combine(iu, bl, ml)
    i3 = combine(i2, bs, ms)
    return dict(bs=bs, bl=bl, bu=bu, ms=ms, ml_sobel=ml0, mx=mx, mn=mn, ml=ml,
                iu=iu, i2=i2, i3=i3)
