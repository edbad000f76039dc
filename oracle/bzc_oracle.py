"""CPU oracle for the PyBlaz (arXiv 2406.11209) compress / compressed-op path.

TEST INFRASTRUCTURE ONLY.  This module is a plain-numpy restatement of the
reference package ``bzc`` (``/root/reference/pkg/src/bzc``) for the hot path
named in BASELINE.json.  It exists so that

* ``tests/`` can check the CUDA path against an independent CPU computation,
* ``__graft_entry__.smoke()`` can check one small CUDA call,
* ``bench.py`` can time a CPU baseline (``cpu_baseline`` / ``--impl reference``).

Nothing in the product package (``paper_2406_11209_b200``) imports this file;
the product path fails loudly when its CUDA library is missing.

Parity of this restatement is pinned against golden vectors produced by the
real reference (``tests/golden/make_golden.py`` imports ``bzc`` from
``/root/reference/pkg/src`` and writes ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.

Representation: every array is a numpy ndarray.  Maxima are held as float64
values that are exactly representable in the float kind (the reference stores
them in the native dtype, ``codec.py:200-206``; widening is exact).  Kinds are
the reference's short names: float kinds ``bf16 f16 f32 f64``
(``kinds.py:30-36``), index kinds ``i8 i16 i32 i64`` (``kinds.py:115-121``).
"""

from __future__ import annotations

import math

import numpy as np

# (stored significand bits, exponent bits) -- kinds.py:84-89
FLOAT_FORMATS = {"bf16": (7, 8), "f16": (10, 5), "f32": (23, 8), "f64": (52, 11)}
INDEX_BITS = {"i8": 8, "i16": 16, "i32": 32, "i64": 64}
INDEX_DTYPES = {"i8": np.int8, "i16": np.int16, "i32": np.int32, "i64": np.int64}


# ---------------------------------------------------------------- kinds ----

def radius(index_kind: str) -> int:
    """r = 2**(b-1) - 1  (kinds.py:128-130)."""
    return (1 << (INDEX_BITS[index_kind] - 1)) - 1


def clamp_bound(index_kind: str) -> float:
    """Largest float64 <= r (kinds.py:137-147): 2**63-1024 for i64."""
    r = radius(index_kind)
    f = float(r)
    if f > r:
        f = math.nextafter(f, 0.0)
    return f


def round_to_kind(x, kind: str) -> np.ndarray:
    """IEEE round-to-nearest-even of float64 values into `kind`.

    Restates kinds.py:186-206: quantum = 2**(max(e-1, emin) - sig) where
    |x| = m * 2**e, m in [0.5, 1); overflow past max_finite gives signed
    infinity; NaN, +-inf and +-0 pass through.  Returns a new float64 array.
    """
    x = np.array(x, dtype=np.float64, copy=True)
    if kind == "f64":
        return x
    sig, ebits = FLOAT_FORMATS[kind]
    emax = (1 << (ebits - 1)) - 1
    emin = 1 - emax
    max_finite = (2.0 - 2.0 ** (-sig)) * 2.0 ** emax
    sel = np.isfinite(x) & (x != 0.0)
    v = x[sel]
    _, e = np.frexp(v)
    qexp = np.maximum(e - 1, emin) - sig
    r = np.ldexp(np.rint(np.ldexp(v, -qexp)), qexp)
    over = np.abs(r) > max_finite
    r[over] = np.copysign(np.inf, v[over])
    x[sel] = r
    return x


# --------------------------------------------------------------- blocking ----

def grid_shape(shape, block_shape):
    """ceil(s / i) per axis (arrays.py:46-48)."""
    return tuple(-(-int(s) // int(b)) for s, b in zip(shape, block_shape))


def block(values: np.ndarray, block_shape) -> np.ndarray:
    """Zero-pad to grid*i and regroup to (grid..., block...) (arrays.py:156-178)."""
    values = np.asarray(values, dtype=np.float64)
    d = values.ndim
    grid = grid_shape(values.shape, block_shape)
    padded = np.zeros(tuple(g * b for g, b in zip(grid, block_shape)))
    padded[tuple(slice(0, s) for s in values.shape)] = values
    split = []
    for g, b in zip(grid, block_shape):
        split += [g, b]
    perm = [2 * k for k in range(d)] + [2 * k + 1 for k in range(d)]
    return np.ascontiguousarray(padded.reshape(split).transpose(perm))


def unblock(blocks: np.ndarray, original_shape) -> np.ndarray:
    """Inverse of :func:`block` followed by the crop (arrays.py:181-190)."""
    d = len(original_shape)
    grid, bshape = blocks.shape[:d], blocks.shape[d:]
    perm = []
    for k in range(d):
        perm += [k, d + k]
    merged = blocks.transpose(perm).reshape(tuple(g * b for g, b in zip(grid, bshape)))
    return np.ascontiguousarray(merged[tuple(slice(0, s) for s in original_shape)])


# ------------------------------------------------------------- transforms ----

def dct_matrix(size: int) -> np.ndarray:
    """Orthonormal DCT-II entries [sample n, basis k] (transforms.py:67-71).

    Evaluated with the same float64 expression as the reference so that the
    entries are bit-identical: sqrt((1+(k>0))/s) * cos(pi*k*(2n+1)/(2s)).
    """
    # vectorised like the reference: numpy's array cos may differ from its
    # scalar cos by an ulp, and the entries must match bit for bit.
    samples = np.arange(size, dtype=np.float64).reshape(size, 1)
    basis = np.arange(size, dtype=np.float64).reshape(1, size)
    scale = np.sqrt(np.where(basis > 0, 2.0, 1.0) / size)
    return scale * np.cos(np.pi * basis * (2.0 * samples + 1.0) / (2.0 * size))


def haar_matrix(size: int) -> np.ndarray:
    """Orthonormal Haar basis, coarse columns first (transforms.py:74-81).

    Column 0 is the scaling vector; then, level by level (coarsest first),
    the wavelets of support size/2**lvl.  An entry that went through t
    halvings of the support carries +-(1/sqrt2)^t, computed as t repeated
    IEEE divisions by sqrt(2) -- the same rounding sequence as the
    reference's recursive construction, hence bit-identical entries.
    """
    levels = int(round(math.log2(size)))
    root2 = np.sqrt(2.0)
    mag = [1.0]
    for _ in range(levels):
        mag.append(mag[-1] / root2)
    h = np.zeros((size, size))
    h[:, 0] = mag[levels]
    col = 1
    for lvl in range(levels):          # lvl 0 = coarsest wavelets
        count = 1 << lvl
        half = size // count // 2      # rows per half-support
        t = levels - lvl               # divisions applied to this level's entries
        for j in range(count):
            for row in range(size):
                coarse = row // half   # row at the level where the wavelet was born
                lower = coarse & 1     # second half of a (+, -) pair
                value = mag[t] if (coarse >> 1) == j else 0.0
                # zeros from the negative half keep their sign (-0.0), as the
                # reference's kron(eye, [[1], [-1]]) produces them
                h[row, col] = -value if lower else value
            col += 1
    return h


def matrix(size: int, family: str) -> np.ndarray:
    return dct_matrix(size) if family == "dct" else haar_matrix(size)


def forward_transform(blocks: np.ndarray, mats) -> np.ndarray:
    """C[..k..] = sum_n B[..n..] H[n,k] along every block axis (transforms.py:118-134)."""
    d = len(mats)
    out = np.asarray(blocks, dtype=np.float64)
    for k, h in enumerate(mats):
        ax = out.ndim - d + k
        out = np.moveaxis(np.moveaxis(out, ax, -1) @ h, -1, ax)
    return np.ascontiguousarray(out)


def inverse_transform(coeffs: np.ndarray, mats) -> np.ndarray:
    """B[..n..] = sum_k C[..k..] H[n,k] along every block axis (transforms.py:137-142)."""
    d = len(mats)
    out = np.asarray(coeffs, dtype=np.float64)
    for k, h in enumerate(mats):
        ax = out.ndim - d + k
        out = np.moveaxis(np.moveaxis(out, ax, -1) @ h.T, -1, ax)
    return np.ascontiguousarray(out)


# ------------------------------------------------------------------ codec ----

def bin_coefficients(coeffs: np.ndarray, d: int, index_kind: str, float_kind: str):
    """(maxima, indices) per codec.py:253-278.

    N = max|C| over the block axes (NaN-propagating), stored rounded into the
    float kind; q = C / N (IEEE f64 division), non-finite q -> 0, then
    clip(rint(q * r), +-clamp_bound).
    """
    axes = tuple(range(coeffs.ndim - d, coeffs.ndim))
    n = round_to_kind(np.max(np.abs(coeffs), axis=axes), float_kind)
    with np.errstate(all="ignore"):
        q = coeffs / n.reshape(n.shape + (1,) * d)
    q = np.where(np.isfinite(q), q, 0.0)
    b = clamp_bound(index_kind)
    idx = np.clip(np.rint(q * float(radius(index_kind))), -b, b)
    return n, idx.astype(INDEX_DTYPES[index_kind])


def kept_positions(mask_bits: np.ndarray) -> np.ndarray:
    """Row-major flat positions of kept coefficients (codec.py:89-92)."""
    return np.flatnonzero(np.asarray(mask_bits, dtype=bool).reshape(-1))


def prune_and_flatten(indices: np.ndarray, mask_bits: np.ndarray) -> np.ndarray:
    """Gather kept positions row-major (codec.py:281-297)."""
    d = mask_bits.ndim
    grid = indices.shape[: indices.ndim - d]
    flat = indices.reshape(grid + (-1,))
    return np.ascontiguousarray(flat[..., kept_positions(mask_bits)])


def unflatten(flat: np.ndarray, mask_bits: np.ndarray) -> np.ndarray:
    """Scatter kept indices back, zeros elsewhere (codec.py:300-318)."""
    grid = flat.shape[:-1]
    full = np.zeros(grid + (mask_bits.size,), dtype=flat.dtype)
    full[..., kept_positions(mask_bits)] = flat
    return full.reshape(grid + mask_bits.shape)


class Settings:
    """Block shape, float kind, index kind, transform family, mask (codec.py:133-179)."""

    def __init__(self, block_shape, float_kind="f32", index_kind="i16",
                 transform="dct", mask_bits=None):
        self.block_shape = tuple(int(b) for b in block_shape)
        self.float_kind = float_kind
        self.index_kind = index_kind
        self.transform = transform
        if mask_bits is None:
            mask_bits = np.ones(self.block_shape, dtype=bool)
        self.mask_bits = np.asarray(mask_bits, dtype=bool).reshape(self.block_shape)

    @property
    def ndim(self):
        return len(self.block_shape)

    @property
    def block_size(self):
        return int(np.prod(self.block_shape))

    @property
    def kept(self):
        return int(self.mask_bits.sum())

    @property
    def keeps_first(self):
        return bool(self.mask_bits.reshape(-1)[0])

    def matrices(self):
        return [matrix(b, self.transform) for b in self.block_shape]


class Compressed:
    """{original shape, settings, maxima (f64 values of the kind), indices} (codec.py:182-223)."""

    def __init__(self, shape, settings: Settings, maxima, indices):
        self.shape = tuple(int(s) for s in shape)
        self.settings = settings
        self.maxima = np.asarray(maxima, dtype=np.float64)
        self.indices = np.asarray(indices)

    @property
    def block_count(self):
        return int(np.prod(self.maxima.shape))


def coefficients(values: np.ndarray, settings: Settings) -> np.ndarray:
    """Transform coefficients of the converted, blocked input (codec.py:327-329)."""
    lowered = round_to_kind(values, settings.float_kind)
    return forward_transform(block(lowered, settings.block_shape), settings.matrices())


def compress(values: np.ndarray, settings: Settings) -> Compressed:
    """convert -> block -> transform -> bin -> prune (codec.py:321-334)."""
    values = np.asarray(values, dtype=np.float64)
    c = coefficients(values, settings)
    n, idx = bin_coefficients(c, settings.ndim, settings.index_kind, settings.float_kind)
    return Compressed(values.shape, settings, n, prune_and_flatten(idx, settings.mask_bits))


def specified_coefficients(a: Compressed) -> np.ndarray:
    """(F * N) / r in f64, multiply before divide (codec.py:337-350)."""
    s = a.settings
    out = unflatten(a.indices, s.mask_bits).astype(np.float64)
    out = out * a.maxima.reshape(a.maxima.shape + (1,) * s.ndim)
    return out / float(radius(s.index_kind))


def decompress(a: Compressed) -> np.ndarray:
    """Inverse transform of the raw indices, then *N, then /r, crop (codec.py:364-384)."""
    s = a.settings
    ints = unflatten(a.indices, s.mask_bits).astype(np.float64)
    blocks = inverse_transform(ints, s.matrices())
    blocks = blocks * a.maxima.reshape(a.maxima.shape + (1,) * s.ndim)
    blocks = blocks / float(radius(s.index_kind))
    return unblock(blocks, a.shape)


# -------------------------------------------------------------------- ops ----

def _rebin(a: Compressed, coeffs: np.ndarray) -> Compressed:
    """Re-quantise with the LEFT operand's settings (ops.py:178-192)."""
    s = a.settings
    n, idx = bin_coefficients(coeffs, s.ndim, s.index_kind, s.float_kind)
    return Compressed(a.shape, s, n, prune_and_flatten(idx, s.mask_bits))


def negate(a: Compressed) -> Compressed:
    """ops.py:195-197."""
    return Compressed(a.shape, a.settings, a.maxima, -a.indices)


def add(a: Compressed, b: Compressed) -> Compressed:
    """ops.py:200-204."""
    return _rebin(a, specified_coefficients(a) + specified_coefficients(b))


def subtract(a: Compressed, b: Compressed) -> Compressed:
    """add(a, negate(b)) -- the reference's subtraction (cli.py:242)."""
    return add(a, negate(b))


def add_scalar(a: Compressed, x: float) -> Compressed:
    """Shift each block's first coefficient by x*sqrt(prod i), rebin (ops.py:207-215)."""
    c = specified_coefficients(a)
    first = (Ellipsis,) + (0,) * a.settings.ndim
    c[first] += float(x) * math.sqrt(a.settings.block_size)
    return _rebin(a, c)


def mul_scalar(a: Compressed, x: float) -> Compressed:
    """N' = RN_kind(N*|x|), F' = F*sign(x) (ops.py:218-223)."""
    x = float(x)
    n = round_to_kind(a.maxima * abs(x), a.settings.float_kind)
    sign = 1 if x > 0 else (-1 if x < 0 else 0)
    return Compressed(a.shape, a.settings, n, (a.indices * sign).astype(a.indices.dtype))


def _products(a: Compressed) -> np.ndarray:
    """F * N per kept coefficient, shape (blocks, kept) (ops.py:144-163)."""
    k = a.settings.kept
    return a.indices.reshape(-1, k).astype(np.float64) * a.maxima.reshape(-1, 1)


def _firsts(a: Compressed) -> np.ndarray:
    """N * F[...,0] / r per block (ops.py:166-175)."""
    f0 = a.indices.reshape(-1, a.settings.kept)[:, 0].astype(np.float64)
    return f0 * a.maxima.reshape(-1) / float(radius(a.settings.index_kind))


def dot(a: Compressed, b: Compressed) -> float:
    """sum(Pa*Pb) / (ra*rb) (ops.py:226-241)."""
    if a.settings.kept == 0:
        return 0.0
    total = float(np.dot(_products(a).ravel(), _products(b).ravel()))
    return total / (float(radius(a.settings.index_kind)) * float(radius(b.settings.index_kind)))


def l2_norm(a: Compressed) -> float:
    """sqrt(sum P^2) / r (ops.py:291-297)."""
    if a.settings.kept == 0:
        return 0.0
    p = _products(a).ravel()
    return float(np.sqrt(float(np.dot(p, p)))) / float(radius(a.settings.index_kind))


def mean(a: Compressed, padding_corrected: bool = False) -> float:
    """ops.py:244-257."""
    f = _firsts(a)
    c = math.sqrt(a.settings.block_size)
    if padding_corrected:
        return float(c * np.sum(f) / np.prod(a.shape))
    return float(np.mean(f) / c)


def covariance(a: Compressed, b: Compressed) -> float:
    """Population covariance over the padded count, DC centred (ops.py:260-283)."""
    nb = a.block_count
    ra = float(radius(a.settings.index_kind))
    rb = float(radius(b.settings.index_kind))
    ma = float(np.sum(_firsts(a)) / nb) * ra
    mb = float(np.sum(_firsts(b)) / nb) * rb
    pa = _products(a)
    pb = _products(b)
    pa[:, 0] -= ma
    pb[:, 0] -= mb
    total = float(np.dot(pa.ravel(), pb.ravel()))
    return total / (ra * rb) / (nb * a.settings.block_size)


def variance(a: Compressed) -> float:
    """ops.py:286-288."""
    return covariance(a, a)


def cosine_similarity(a: Compressed, b: Compressed) -> float:
    """ops.py:300-306 (raises ZeroDivisionError-free ValueError on zero norm)."""
    na, nb = l2_norm(a), l2_norm(b)
    if na == 0.0 or nb == 0.0:
        raise ValueError("zero norm operand")
    return dot(a, b) / (na * nb)


def ssim_components(a: Compressed, b: Compressed, sl=1e-4, sc=9e-4):
    """Luminance, contrast, structure (ops.py:317-335)."""
    mu_a, mu_b = mean(a), mean(b)
    va, vb = variance(a), variance(b)
    sa, sb = math.sqrt(va), math.sqrt(vb)
    cov = covariance(a, b)
    lum = (2 * mu_a * mu_b + sl) / (mu_a * mu_a + mu_b * mu_b + sl)
    con = (2 * sa * sb + sc) / (va + vb + sc)
    st = (cov + sc / 2) / (sa * sb + sc / 2)
    return lum, con, st


def ssim(a: Compressed, b: Compressed, sl=1e-4, sc=9e-4, wl=1.0, wc=1.0, ws=1.0) -> float:
    """Weighted product of the three terms (ops.py:338-348)."""
    lum, con, st = ssim_components(a, b, sl, sc)
    return float(lum) ** wl * float(con) ** wc * float(st) ** ws


def gradient_array(shape) -> np.ndarray:
    """X[x] = sum(x) / sum(s - 1) (arrays.py:193-208), float64 values."""
    shape = tuple(int(s) for s in shape)
    total = np.zeros(shape)
    for ax, n in enumerate(shape):
        view = [1] * len(shape)
        view[ax] = n
        total = total + np.arange(n, dtype=np.float64).reshape(view)
    return total / sum(s - 1 for s in shape)


# ---------------------------------------------------------- tie handling ----

def tie_mask(coeffs: np.ndarray, maxima: np.ndarray, d: int, index_kind: str,
             window: float = 2.0 ** -36) -> np.ndarray:
    """Coefficients whose pre-rounding bin value sits near a half-integer.

    v = (C / N) * r is the value the reference rounds (codec.py:272-277).
    Two implementations that compute C in different (equally valid) f64
    summation orders can round such v differently; SURVEY.md §7.1 calls
    these ties.  Returns a bool mask shaped like `coeffs`.
    """
    with np.errstate(all="ignore"):
        v = coeffs / maxima.reshape(maxima.shape + (1,) * d) * float(radius(index_kind))
    v = np.where(np.isfinite(v), v, 0.0)
    frac = np.abs(v - np.floor(v) - 0.5)
    return frac <= window * np.maximum(1.0, np.abs(v))
