"""numpy restatement of the GPU synth_pair's closed-form recipe (csrc/synth.cu).

TEST INFRASTRUCTURE: the CPU side of SURVEY 8(d)'s spot check of the GPU
generator (the bench's and config 5's inputs come from it).  SPEC.md:415-423:
F = Gaussian blobs normalised to [0, 1] (+ N(0, noise^2)); u_true = a
Gaussian-smoothed N(0, 1) field scaled to max |u| = warp_max; M = clean F
sampled at x + u_true (+ independent noise).  The random numbers are the
generator's counter-based SplitMix64 hash, so every voxel is computable on
its own.
"""
import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uni(seed, stream, i):
    with np.errstate(over="ignore"):
        inner = np.uint64(stream) * np.uint64(0x632BE59BD9B4E019) + np.asarray(i, np.uint64)
    return (mix64(np.uint64(seed) ^ mix64(inner)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def normal(seed, stream, i):
    i = np.asarray(i, np.uint64)
    u1 = 1.0 - uni(seed, stream, np.uint64(2) * i)
    u2 = uni(seed, stream, np.uint64(2) * i + np.uint64(1))
    return (np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)).astype(np.float32)


def blobs(shape, seed, num_blobs):
    """Host-side blob parameters: serial SplitMix64 from the seed."""
    nz, ny, nx = shape
    state = int(seed)
    out = []

    def u01():
        nonlocal state
        r = int(mix64(np.uint64(state & 0xFFFFFFFFFFFFFFFF)))
        state += 1
        return (r >> 11) * 2.0 ** -53

    mind = float(min(nx, ny, nz))
    for _ in range(num_blobs):
        cx = np.float32((0.2 + 0.6 * u01()) * nx)
        cy = np.float32((0.2 + 0.6 * u01()) * ny)
        cz = np.float32((0.2 + 0.6 * u01()) * nz)
        sg = (0.05 + 0.07 * u01()) * mind
        q = np.float32(1.0 / (2.0 * sg * sg))
        amp = np.float32(0.3 + 0.7 * u01())
        out.append((cx, cy, cz, q, amp))
    return out


def clean_fixed(shape, seed, num_blobs):
    """Blob image (fp32 sum in blob order), min-max normalised."""
    nz, ny, nx = shape
    z, y, x = np.meshgrid(np.arange(nz, dtype=np.float32), np.arange(ny, dtype=np.float32),
                          np.arange(nx, dtype=np.float32), indexing="ij")
    s = np.zeros(shape, np.float32)
    for cx, cy, cz, q, amp in blobs(shape, seed, num_blobs):
        dx, dy, dz = x - cx, y - cy, z - cz
        s = s + amp * np.exp(-(dx * dx + dy * dy + dz * dz) * q).astype(np.float32)
    lo, hi = s.min(), s.max()
    inv = np.float32(1.0) / (hi - lo) if hi > lo else np.float32(1.0)
    return ((s - lo) * inv).astype(np.float32)


def smooth_axis(a, axis, sigma):
    """k_smooth_axis: fp32 taps truncated at max(1, ceil(3 sigma)),
    renormalised over in-bounds taps."""
    R = max(1, int(np.ceil(3.0 * sigma)))
    w = np.exp(-0.5 * np.arange(-R, R + 1, dtype=np.float64) ** 2 / sigma ** 2).astype(np.float32)
    n = a.shape[axis]
    a = np.moveaxis(a, axis, -1)
    num = np.zeros_like(a)
    den = np.zeros(n, np.float32)
    for t in range(-R, R + 1):
        lo, hi = max(0, -t), min(n, n - t)
        num[..., lo:hi] = (num[..., lo:hi] + w[t + R] * a[..., lo + t:hi + t]).astype(np.float32)
        den[lo:hi] += w[t + R]
    return np.moveaxis((num / den).astype(np.float32), -1, axis)


def true_warp(shape, seed, warp_max, attempt=0, warp_sigma=0.0):
    """u_true as (3, nz, ny, nx): N(0,1) per component (stream 7 + attempt),
    smoothed x, y, z, scaled so that max |u| = warp_max."""
    n = int(np.prod(shape))
    U = normal(seed, 7 + attempt, np.arange(3 * n, dtype=np.uint64)).reshape((3,) + tuple(shape))
    ws = warp_sigma if warp_sigma > 0 else min(shape) / 16.0
    ws = min(ws, 21.0)
    S = U
    for ax in (3, 2, 1):
        S = smooth_axis(S, ax, ws)
    m = np.abs(S).max()
    return (S * np.float32(warp_max / m if m > 0 else 0.0)).astype(np.float32)


def sample_exact(Fc, u, idx):
    """Fc sampled at voxel idx + u (fp64 lerps of the fp32 image, rounded
    once), field.cpp's clamp rules; idx: flat voxel indices."""
    nz, ny, nx = Fc.shape
    z, y, x = np.unravel_index(idx, Fc.shape)
    ux, uy, uz = (u[c].reshape(-1)[idx] for c in range(3))

    def axis(p, d, n):
        c = p.astype(np.float64) + d.astype(np.float64)
        c = np.clip(c, 0.0, n - 1.0)
        i0 = np.minimum(np.floor(c), n - 2).astype(np.int64)
        t = c - i0
        return np.maximum(i0, 0), t

    x0, tx = axis(x, ux, nx)
    y0, ty = axis(y, uy, ny)
    z0, tz = axis(z, uz, nz)
    V = Fc.astype(np.float64)

    def at(dx, dy, dz):
        return V[np.minimum(z0 + dz, nz - 1), np.minimum(y0 + dy, ny - 1), np.minimum(x0 + dx, nx - 1)]

    v00 = at(0, 0, 0) + tx * (at(1, 0, 0) - at(0, 0, 0))
    v10 = at(0, 1, 0) + tx * (at(1, 1, 0) - at(0, 1, 0))
    v01 = at(0, 0, 1) + tx * (at(1, 0, 1) - at(0, 0, 1))
    v11 = at(0, 1, 1) + tx * (at(1, 1, 1) - at(0, 1, 1))
    s0 = v00 + ty * (v10 - v00)
    s1 = v01 + ty * (v11 - v01)
    return (s0 + tz * (s1 - s0)).astype(np.float32)
