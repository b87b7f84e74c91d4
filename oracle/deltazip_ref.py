"""numpy float64 restatement of the DeltaZip hot path (test oracle, not product).

Every function cites the reference location it restates. The arithmetic is
the reference's: f64 everywhere, codes decoded without clamping, scales
widened from f32, dense GEMVs via numpy `@`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SPARSITY_NONE = "none"            # compress.py:32
SPARSITY_2_4 = "two_of_four"      # compress.py:33
AXIS_COLUMN = "column"            # core.py:18
AXIS_ROW = "row"                  # core.py:19
VALID_BITS = (2, 3, 4, 8, 16)     # compress.py:38


class OracleError(Exception):
    """Raised where the reference raises a DeltaZipError; `kind` names the class."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


@dataclass
class OracleDelta:
    """Field-for-field mirror of `LayerDelta` (compress.py:101-143)."""

    rows: int
    cols: int
    packed_values: np.ndarray   # <u4
    index_stream: bytes
    scales: np.ndarray          # <f4
    bits: int
    sparsity: str
    group_size: int
    name: str = "layer"

    @property
    def n_groups(self) -> int:  # compress.py:141-143
        return math.ceil(self.cols / self.group_size)


def _qmax(bits: int) -> int:
    return (1 << (bits - 1)) - 1


# --------------------------------------------------------------------------- codec


def pack_codes(codes, bits: int) -> np.ndarray:
    """compress.py:243-262 — offset-unsigned codes, LSB first, 32//bits per word."""
    if not 2 <= bits <= 16:
        raise ValueError(f"bits must be in [2, 16], got {bits}")
    c = np.asarray(codes, dtype=np.int64).ravel()
    q = _qmax(bits)
    if c.size and (int(c.min()) < -q or int(c.max()) > q):
        raise OracleError("EncodingError", "code out of range")
    per = 32 // bits
    nw = -(-c.size // per)
    u = np.zeros(nw * per, dtype=np.uint64)
    u[: c.size] = (c + q).astype(np.uint64)
    words = np.zeros(nw, dtype=np.uint64)
    for j in range(per):
        words |= u[j::per] << np.uint64(bits * j)
    return (words & np.uint64(0xFFFFFFFF)).astype("<u4")


def unpack_codes(words, bits: int, count: int) -> np.ndarray:
    """compress.py:265-277 — no clamping: u - qmax for any u."""
    if not 2 <= bits <= 16:
        raise ValueError(f"bits must be in [2, 16], got {bits}")
    w = np.asarray(words, dtype=np.uint32).astype(np.uint64)
    per = 32 // bits
    if count > w.size * per:
        raise OracleError("EncodingError", f"cannot unpack {count} codes from {w.size} words")
    mask = np.uint64((1 << bits) - 1)
    out = np.empty((w.size, per), dtype=np.int64)
    for j in range(per):
        out[:, j] = ((w >> np.uint64(bits * j)) & mask).astype(np.int64)
    return out.ravel()[:count] - _qmax(bits)


def encode_mask_indices(keep: np.ndarray) -> bytes:
    """compress.py:280-292 — one nibble (p0 | p1<<2) per 4-col group, low nibble first."""
    keep = np.asarray(keep, dtype=bool)
    rows, cols = keep.shape
    g = keep.reshape(-1, 4)
    pos = np.argwhere(g)[:, 1].reshape(-1, 2)
    nib = (pos[:, 0] | (pos[:, 1] << 2)).astype(np.uint8)
    if nib.size % 2:
        nib = np.concatenate([nib, np.zeros(1, np.uint8)])
    return (nib[0::2] | (nib[1::2] << 4)).astype(np.uint8).tobytes()


def decode_mask_indices(data: bytes, rows: int, cols: int) -> np.ndarray:
    """compress.py:295-314 — length check and p0<p1 check raise FormatError."""
    n = rows * (cols // 4)
    if len(data) != -(-n // 2):
        raise OracleError("FormatError", f"index stream length {len(data)} != {-(-n // 2)}")
    raw = np.frombuffer(bytes(data), dtype=np.uint8)
    nib = np.empty(raw.size * 2, dtype=np.uint8)
    nib[0::2] = raw & 0xF
    nib[1::2] = raw >> 4
    nib = nib[:n]
    p0, p1 = nib & 3, nib >> 2
    if np.any(p0 >= p1):
        raise OracleError("FormatError", "kept positions not strictly increasing")
    keep = np.zeros((n, 4), dtype=bool)
    keep[np.arange(n), p0] = True
    keep[np.arange(n), p1] = True
    return keep.reshape(rows, cols)


def float64_unpayload(words, count: int) -> np.ndarray:
    """compress.py:343-345 — bits=16 passthrough: raw little-endian f64 in u32 pairs."""
    return np.frombuffer(np.ascontiguousarray(words, dtype="<u4").tobytes(), dtype="<f8")[:count].copy()


def float64_payload(values) -> np.ndarray:
    """compress.py:339-340."""
    return np.frombuffer(np.ascontiguousarray(values, dtype="<f8").tobytes(), dtype="<u4").copy()


def dequantize_layer(ld) -> np.ndarray:
    """compress.py:467-497 — dense f64 ΔW[r,c] = code * scale[r, c//gs] at kept positions."""
    r, c = int(ld.rows), int(ld.cols)
    sparse = ld.sparsity == SPARSITY_2_4
    keep = decode_mask_indices(ld.index_stream, r, c) if sparse else None
    n = r * c // 2 if sparse else r * c
    scales = np.asarray(ld.scales, dtype="<f4")
    if ld.bits == 16 and scales.size == 0:
        vals = float64_unpayload(ld.packed_values, n)
    else:
        codes = unpack_codes(ld.packed_values, ld.bits, n).astype(np.float64)
        ng = -(-c // ld.group_size)
        grid = scales.astype(np.float64).reshape(r, ng)  # wrong length -> numpy ValueError, as ref
        per = grid[:, np.arange(c) // ld.group_size]
        if not sparse:
            return codes.reshape(r, c) * per
        vals = codes * per[keep]
    out = np.zeros((r, c), dtype=np.float64)
    if sparse:
        out[keep] = vals
    else:
        out[:] = vals.reshape(r, c)
    return out


# --------------------------------------------------------------------------- serving math


def as_matrix(a) -> np.ndarray:
    """core.py:22-29."""
    m = np.ascontiguousarray(a, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] < 1 or m.shape[1] < 1:
        raise OracleError("ShapeError", f"bad matrix shape {m.shape}")
    return m


def decoupled_linear(w_base, ld, x) -> np.ndarray:
    """inference.py:94-103 — W_base @ x + dequant(ΔW) @ x, never merged."""
    w = as_matrix(w_base)
    if (ld.rows, ld.cols) != w.shape:
        raise OracleError("ShapeError", "delta/base shape mismatch")
    xm = np.asarray(x, dtype=np.float64)
    vec = xm.ndim == 1
    if vec:
        xm = xm.reshape(-1, 1)
    if xm.ndim != 2 or xm.shape[0] != w.shape[1]:
        raise OracleError("ShapeError", "input shape")
    out = w @ xm + dequantize_layer(ld) @ xm
    return out[:, 0] if vec else out


def group_by_delta(delta_ids):
    """inference.py:106-123 — stable sort by delta id; perm[orig] = sorted position."""
    ids = [int(d) for d in delta_ids]
    order = sorted(range(len(ids)), key=lambda i: ids[i])
    perm = [0] * len(ids)
    groups = []
    for pos, orig in enumerate(order):
        perm[orig] = pos
        if groups and groups[-1][0] == ids[orig]:
            groups[-1] = (ids[orig], groups[-1][1], pos + 1)
        else:
            groups.append((ids[orig], pos, pos + 1))
    return perm, groups


def sbmm(base_layer, deltas, rows) -> dict:
    """inference.py:126-154 — rows: list of (request_id, delta_id, x).

    UnknownDeltaError before compute; each delta dequantised once per call;
    outputs keyed by request id in original order (last duplicate wins).
    """
    w = as_matrix(base_layer)
    for rid, did, _ in rows:
        if did not in deltas:
            raise OracleError("UnknownDeltaError", f"request {rid}: delta {did}")
    perm, groups = group_by_delta([d for _, d, _ in rows])
    order = [0] * len(perm)
    for orig, pos in enumerate(perm):
        order[pos] = orig
    out = {}
    for did, s, e in groups:
        dq = dequantize_layer(deltas[did])
        if dq.shape != w.shape:
            raise OracleError("ShapeError", f"delta {did} shape {dq.shape} != base {w.shape}")
        for pos in range(s, e):
            rid, _, x = rows[order[pos]]
            x = np.asarray(x, dtype=np.float64).ravel()
            out[rid] = w @ x + dq @ x
    return {rid: out[rid] for rid, _, _ in rows}


def sbmm_matrix(base_layer, deltas, delta_ids, X) -> np.ndarray:
    """Batched restatement of `sbmm` for throughput baselines: X[T, in] -> Y[T, out].

    Same per-delta dequantise-once structure (inference.py:145-153); the per-row
    GEMVs of one group are issued as one numpy GEMM over that group's rows.
    """
    w = as_matrix(base_layer)
    X = np.asarray(X, dtype=np.float64)
    ids = np.asarray(delta_ids)
    Y = np.empty((X.shape[0], w.shape[0]), dtype=np.float64)
    for did in sorted(set(ids.tolist())):
        sel = np.nonzero(ids == did)[0]
        dq = dequantize_layer(deltas[did])
        xs = X[sel]
        Y[sel] = xs @ w.T + xs @ dq.T
    return Y


def tp_partition(w, axis: str, n: int):
    """inference.py:162-177 — contiguous column / row blocks (copies)."""
    w = as_matrix(w)
    if n < 1:
        raise OracleError("PartitionError", "n < 1")
    if axis == AXIS_COLUMN:
        if w.shape[1] % n:
            raise OracleError("PartitionError", "columns not divisible")
        s = w.shape[1] // n
        return [w[:, i * s:(i + 1) * s].copy() for i in range(n)]
    if axis == AXIS_ROW:
        if w.shape[0] % n:
            raise OracleError("PartitionError", "rows not divisible")
        s = w.shape[0] // n
        return [w[i * s:(i + 1) * s, :].copy() for i in range(n)]
    raise OracleError("PartitionError", f"axis {axis!r}")


def tp_forward(base_shards, delta_shards, x, axis: str) -> np.ndarray:
    """inference.py:180-225 — column: concat of shard outputs; row: shard-order partial sum."""
    if len(base_shards) != len(delta_shards):
        raise OracleError("PartitionError", "shard count mismatch")
    x = as_matrix(x)
    for b, d in zip(base_shards, delta_shards):
        if b.shape != d.shape:
            raise OracleError("PartitionError", "shard shape mismatch")
    if axis == AXIS_COLUMN:
        if x.shape[1] != base_shards[0].shape[0]:
            raise OracleError("PartitionError", "activation dim")
        return np.concatenate([x @ b + x @ d for b, d in zip(base_shards, delta_shards)], axis=1)
    if axis == AXIS_ROW:
        if x.shape[1] != sum(b.shape[0] for b in base_shards):
            raise OracleError("PartitionError", "activation dim")
        out, start = None, 0
        for b, d in zip(base_shards, delta_shards):
            xs = x[:, start:start + b.shape[0]]
            start += b.shape[0]
            part = xs @ b + xs @ d
            out = part if out is None else out + part
        return out
    raise OracleError("PartitionError", f"axis {axis!r}")


def forward_model(base_layers, deltas_per_id, rows):
    """inference.py:246-291 (no-TP branch) — per-layer sbmm, tanh between layers.

    base_layers: list of W (out, in); deltas_per_id: {did: [layer deltas]}.
    """
    cur = {rid: np.asarray(x, dtype=np.float64).ravel() for rid, _, x in rows}
    nl = len(base_layers)
    for li, w in enumerate(base_layers):
        lrows = [(rid, did, cur[rid]) for rid, did, _ in rows]
        outs = sbmm(w, {did: deltas_per_id[did][li] for _, did, _ in rows}, lrows)
        if li + 1 < nl:
            outs = {k: np.tanh(v) for k, v in outs.items()}
        cur = outs
    return cur


# --------------------------------------------------------------------------- fixtures


def magnitude_rtn_2of4(delta: np.ndarray, bits: int, group_size: int = 128):
    """Synthetic ΔCompress producer following `tests/oracles.py:82-107`
    (magnitude 2:4 prune + symmetric RTN per (row, group), f32 scales), returned
    as an `OracleDelta` in the reference packed layout (compress.py:439-452)."""
    d = np.asarray(delta, dtype=np.float64)
    r, c = d.shape
    q = _qmax(bits)
    keep = np.ones((r, c), dtype=bool)
    for g0 in range(0, c, 4):
        o = np.argsort(np.abs(d[:, g0:g0 + 4]), axis=1, kind="stable")
        keep[np.arange(r), g0 + o[:, 0]] = False
        keep[np.arange(r), g0 + o[:, 1]] = False
    ng = -(-c // group_size)
    scales = np.zeros((r, ng), dtype=np.float64)
    codes = np.zeros((r, c), dtype=np.int64)
    for g in range(ng):
        seg = d[:, g * group_size:(g + 1) * group_size]
        s = np.float64(np.float32(np.max(np.abs(seg), axis=1) / q))
        scales[:, g] = s
        nz = s > 0
        cc = np.zeros_like(seg, dtype=np.int64)
        cc[nz] = np.clip(np.rint(seg[nz] / s[nz, None]), -q, q).astype(np.int64)
        codes[:, g * group_size:(g + 1) * group_size] = cc
    return OracleDelta(
        rows=r, cols=c,
        packed_values=pack_codes(codes[keep], bits),
        index_stream=encode_mask_indices(keep),
        scales=scales.astype("<f4").ravel(),
        bits=bits, sparsity=SPARSITY_2_4, group_size=group_size,
    )


def random_packed_delta(rng: np.random.Generator, rows: int, cols: int, bits: int,
                        group_size: int = 128, sparse: bool = True, scale_std: float = 0.02):
    """Uniform random packed delta (any u in [0, 2^bits) incl. the unclamped
    code qmax+1), random valid nibbles, |N| f32 scales — SURVEY §8(d) recipe."""
    n = rows * cols // 2 if sparse else rows * cols
    per = 32 // bits
    nw = -(-n // per)
    words = rng.integers(0, 2 ** 32, size=nw, dtype=np.uint64).astype("<u4")
    if n % per:  # reference zero-pads the final word (compress.py:256-260)
        keep_bits = (n % per) * bits
        words[-1] &= np.uint32((1 << keep_bits) - 1)
    index = b""
    if sparse:
        nib = np.array([0x4, 0x8, 0xC, 0x9, 0xD, 0xE], dtype=np.uint8)[
            rng.integers(0, 6, size=rows * (cols // 4))]
        if nib.size % 2:
            nib = np.concatenate([nib, np.zeros(1, np.uint8)])
        index = (nib[0::2] | (nib[1::2] << 4)).tobytes()
    ng = -(-cols // group_size)
    scales = (np.abs(rng.normal(0, scale_std, size=rows * ng)) / max(_qmax(bits), 1)).astype("<f4")
    return OracleDelta(rows=rows, cols=cols, packed_values=words, index_stream=index,
                       scales=scales, bits=bits,
                       sparsity=SPARSITY_2_4 if sparse else SPARSITY_NONE, group_size=group_size)


# --------------------------------------------------------------------------- ΔCompress solver
# (the offline producer of packed deltas, restated for the GPU solver's tests)


def compute_hessian(samples: np.ndarray, damping: float) -> np.ndarray:
    """H = X X^T + damping * mean(diag(X X^T)) * I  (compress.py:178-186)."""
    x = np.asarray(samples, dtype=np.float64)
    h = x @ x.T
    h[np.diag_indices_from(h)] += damping * float(np.mean(np.diag(h)))
    return h


def inverse_cholesky_factor(hessian: np.ndarray) -> np.ndarray:
    """Upper U with H^-1 = U^T U (compress.py:321-336), via LAPACK like the reference."""
    import scipy.linalg as sla
    try:
        cf = sla.cho_factor(hessian, lower=True, check_finite=False)
        hinv = sla.cho_solve(cf, np.eye(hessian.shape[0]), check_finite=False)
        return sla.cholesky(hinv, lower=False, check_finite=False)
    except (np.linalg.LinAlgError, sla.LinAlgError, ValueError) as exc:
        raise OracleError("NumericDomainError", f"hessian is not positive definite: {exc}") from exc


def keep_mask_groups(w4: np.ndarray, hd: np.ndarray) -> np.ndarray:
    """2:4 keep-mask per row of 4 (compress.py:204-215): prune the two smallest saliencies
    w^2 / hd, ties to the lower index (stable order)."""
    sal = w4 * w4 / hd
    rank = np.argsort(np.argsort(sal, axis=1, kind="stable"), axis=1, kind="stable")
    return rank >= 2


def obs_compress_layer(delta, hessian, bits: int, sparsity: str, group_size: int, block_size: int,
                       u: np.ndarray | None = None):
    """Greedy OBS column solver (compress.py:348-464). Returns (OracleDelta, proxy_loss,
    quantized dense f64 delta). `u` overrides the inverse-Hessian factor (the GPU tests pass
    the same factor to both sides)."""
    w = np.array(delta, dtype=np.float64)
    r, c = w.shape
    sparse = sparsity == SPARSITY_2_4
    passthrough = bits == 16
    if passthrough and not sparse:  # compress.py:372-385
        return (OracleDelta(rows=r, cols=c, packed_values=float64_payload(w), index_stream=b"",
                            scales=np.zeros(0, "<f4"), bits=bits, sparsity=sparsity,
                            group_size=group_size), 0.0, w.copy())
    if u is None:
        u = inverse_cholesky_factor(np.asarray(hessian, dtype=np.float64))
    ud = np.diag(u)
    q = _qmax(bits)
    ng = -(-c // group_size)
    keep = np.ones((r, c), dtype=bool)
    codes = np.zeros((r, c), dtype=np.int64)
    quant = np.zeros((r, c))
    scales = np.zeros((r, ng))
    loss = 0.0
    for b0 in range(0, c, block_size):
        b1 = min(b0 + block_size, c)
        blk = w[:, b0:b1].copy()            # the in-block working copy (`w1`)
        errs = np.zeros_like(blk)
        for j in range(b1 - b0):
            col = b0 + j
            if not passthrough and col % group_size == 0:   # scale from the block-start `w`
                mx = np.max(np.abs(w[:, col:min(col + group_size, c)]), axis=1)
                scales[:, col // group_size] = (mx / q).astype(np.float32).astype(np.float64)
            if sparse and col % 4 == 0:
                keep[:, col:col + 4] = keep_mask_groups(blk[:, j:j + 4], ud[col:col + 4] ** 2)
            wc, kc = blk[:, j], keep[:, col]
            if passthrough:
                qc = np.where(kc, wc, 0.0)
            else:
                s = scales[:, col // group_size]
                m = kc & (s > 0)
                cc = np.zeros(r, dtype=np.int64)
                cc[m] = np.clip(np.rint(wc[m] / s[m]), -q, q).astype(np.int64)
                codes[:, col] = cc
                qc = cc.astype(np.float64) * s
            quant[:, col] = qc
            e = (wc - qc) / ud[col]
            loss += float(np.sum((wc - qc) ** 2) / (ud[col] * ud[col]))
            blk[:, j + 1:] -= np.outer(e, u[col, col + 1:b1])
            errs[:, j] = e
        w[:, b0:b1] = quant[:, b0:b1]
        if b1 < c:
            w[:, b1:] -= errs @ u[b0:b1, b1:]
    if sparse:
        index = encode_mask_indices(keep)
        packed = float64_payload(quant[keep]) if passthrough else pack_codes(codes[keep], bits)
    else:
        index, packed = b"", pack_codes(codes.reshape(-1), bits)
    sc = np.zeros(0, "<f4") if passthrough else scales.astype("<f4").reshape(-1)
    od = OracleDelta(rows=r, cols=c, packed_values=packed, index_stream=index, scales=sc, bits=bits,
                     sparsity=sparsity, group_size=group_size)
    return od, loss, quant


# --------------------------------------------------------------------------- admission
# (the decision of scheduler.select_batch, scheduler.py:73-123, restated as the
#  checker of the on-device admission kernel; pinned to traces the reference produced,
#  tests/golden/make_admit.py)


def select_batch(queue, running, K: int, N: int):
    """queue / running: lists of (request id, arrival, model id); the queue in (arrival, id) order.
    Returns (batch ids in batch order, {line-skip id: parent id}, selected delta set).
    scheduler.py:84-104: running requests first (sorted by key), then the head-first scan."""
    key = {i: (a, i) for i, a, _ in list(queue) + list(running)}
    selected = {m for _, _, m in running}
    batch = sorted(((i, m) for i, _, m in running), key=lambda r: key[r[0]])
    passed_over = False
    skips = {}
    for i, _, m in queue:
        if len(batch) >= K:
            break
        if m in selected or len(selected) < N:
            if passed_over:
                skips[i] = min((r for r in batch if r[1] == m), key=lambda r: key[r[0]])[0]
            selected.add(m)
            batch.append((i, m))
        else:
            passed_over = True
    return [i for i, _ in batch], skips, selected
