"""Host emulator of a lowered launch plan (TEST INFRASTRUCTURE).

Executes the exact argument blocks `compiler.lower` produces — magic-number
digit maps, VM programs, strides — on numpy buffers, so the fusion and
index-map logic can be checked against the oracle on a GPU-less host.  It
decodes the same `abi` structures the CUDA kernels read.  Reductions fold
sequentially (the reference order), so emulated results are bit-comparable
with the oracle; the GPU's tree orders are checked separately on the box.
"""

from __future__ import annotations

import numpy as np

from paper_1801_08058_b200 import abi
from paper_1801_08058_b200.compiler import decode_flat

DT = {abi.K_EW1_F32: np.float32, abi.K_EW1_F64: np.float64, abi.K_EWS_F32: np.float32, abi.K_EWS_F64: np.float64, abi.K_EW_F32: np.float32, abi.K_EW_F64: np.float64, abi.K_EW_I64: np.int64, abi.K_EW_U8: np.uint8,
      abi.K_DOT_F32: np.float32, abi.K_DOT_F64: np.float64, abi.K_DOT_SM_F32: np.float32, abi.K_DOT_SM_F64: np.float64, abi.K_DOT_TH_F32: np.float32, abi.K_DOT_TH_F64: np.float64, abi.K_CONV_F32: np.float32, abi.K_CONV_F64: np.float64}


def _fdiv(n, mul, sh):
    if mul == 0:
        return n
    return ((n.astype(np.uint64) * np.uint64(mul)) >> np.uint64(32 + sh)).astype(np.int64)


def leaf_offsets(L, o, r):
    if L.rlin >= 0:  # the kernel's fast path must agree with the digits
        rd = [L.dig[i] for i in range(L.ndig) if L.dig[i].src == 1]
        assert (not rd and L.rlin == 0) or (len(rd) == 1 and rd[0].div_mul == 0 and rd[0].mod == 0 and rd[0].stride == L.rlin)
    off = np.zeros_like(o)
    for i in range(L.ndig):
        d = L.dig[i]
        n = r if d.src else o
        q = _fdiv(n, d.div_mul, d.div_sh)
        if d.mod:
            q = q - _fdiv(q, d.mod_mul, d.mod_sh) * d.mod
        off = off + q * d.stride
    return off


class Memory:
    def __init__(self, lowered, inputs, outputs):
        self.slots = {abi.SLOT_ARENA: np.zeros(max(lowered.arena_bytes, 8), dtype=np.uint8),
                      abi.SLOT_CONST: np.frombuffer(lowered.const_blob + b"\0" * 8, dtype=np.uint8).copy()}
        for i, a in enumerate(inputs):
            self.slots[abi.SLOT_IO + i] = a.view(np.uint8).reshape(-1)
        for j, a in enumerate(outputs):
            self.slots[abi.SLOT_IO + len(inputs) + j] = a.view(np.uint8).reshape(-1)

    def view(self, ref, dtype):
        slot, off = ref >> 56, ref & ((1 << 56) - 1)
        raw = self.slots[slot]
        item = np.dtype(dtype).itemsize
        n = (raw.size - off) // item
        return raw[off: off + n * item].view(dtype)


def _un(op, a, dt):
    with np.errstate(all="ignore"):
        if op == 5:
            return (-a).astype(dt) if dt != np.int64 else (np.uint64(0) - a.astype(np.uint64)).astype(np.int64)
        x = a.astype(np.float64)
        if op == 6:
            y = np.exp(x)
        elif op == 7:
            y = np.where(x < 0, np.nan, np.where(x == 0, -np.inf, np.log(np.where(x > 0, x, 1.0))))
            y = np.where(np.isnan(x), x, y)
        elif op == 8:
            y = np.tanh(x)
        elif op == 9:
            pos = 1.0 / (1.0 + np.exp(-np.where(x >= 0, x, 0.0)))
            e = np.exp(np.where(x < 0, x, 0.0))
            y = np.where(x >= 0, pos, e / (1.0 + e))
            y = np.where(np.isnan(x), x, y)
        elif op == 10:
            return np.where(a > 0, a, np.zeros_like(a)).astype(dt)
        else:
            raise ValueError(op)
        return y.astype(dt)


def _bin(op, x, y, dt):
    with np.errstate(all="ignore"):
        if dt == np.int64:
            ux, uy = x.astype(np.uint64), y.astype(np.uint64)
            return {0: ux + uy, 1: ux - uy, 2: ux * uy}[op].astype(np.int64)
        if op == 0:
            return (x + y).astype(dt)
        if op == 1:
            return (x - y).astype(dt)
        if op == 2:
            return (x * y).astype(dt)
        if op == 3:
            return (x / y).astype(dt)
        if op == 4:
            return np.where(x >= y, x, y).astype(dt)
    raise ValueError(op)


def run_ew(mem, a, dt):
    n_o, n_r = a.n_o, a.n_r
    assert a.mode in (1, 2, 3) and a.vec_axis == (0 if a.mode == 2 else 1)
    o = np.repeat(np.arange(n_o, dtype=np.int64), n_r)
    r = np.tile(np.arange(n_r, dtype=np.int64), n_o)

    def load(k):
        L = a.leaves[k]
        if L.mode == 1:
            raw = np.array([L.splat], dtype=np.uint64)
            if dt == np.float32:
                v = raw.astype(np.uint32).view(np.float32)[0]
            elif dt == np.uint8:
                v = np.uint8(L.splat & 0xFF)
            else:
                v = raw.view(dt)[0]
            return np.full(o.shape, v, dtype=dt)
        return mem.view(L.ref, dt)[leaf_offsets(L, o, r)]

    acc = None
    stack = []
    pre = [load(k) for k in range(a.npre)]
    if a.mode == 3:  # the staged kernel only implements these sources
        for pc in range(a.ninstr):
            ins = decode_flat(a.prog[pc])
            assert ins[0] in ("loadp", "store", "un") or (ins[0] == "bin" and ins[1] in (0, 1, 2, 3, 6)), ins
    for pc in range(a.ninstr):
        ins = decode_flat(a.prog[pc])
        if ins[0] == "loadp":
            acc = pre[ins[1]]
        elif ins[0] == "loadm":
            acc = load(ins[1])
        elif ins[0] == "push":
            stack.append(acc)
        elif ins[0] == "store":
            L = a.leaves[ins[1]]
            mem.view(L.ref, dt)[leaf_offsets(L, o, r)] = acc
        elif ins[0] == "un":
            acc = _un(ins[1], acc, dt)
        elif ins[0] == "dot":  # acc = acc + a * b, two roundings
            va, vb = load(ins[1]), load(ins[2])
            acc = _bin(0, acc, _bin(2, va, vb, dt), dt)
        else:
            _, src, op, sw, k = ins
            if src < 4:
                b = pre[src]
            elif src == 4:
                b = load(k)
            elif src == 5:
                b = stack.pop()
            else:
                b = acc
            acc = _bin(op, b, acc, dt) if sw else _bin(op, acc, b, dt)
    if a.red_kind == 0:
        return
    vals = acc.reshape(n_o, n_r) if (acc is not None and n_r) else np.zeros((n_o, 0), dtype=dt)
    if a.red_kind == 2:
        red = np.full(n_o, -np.inf, dtype=dt)
        for j in range(n_r):
            red = np.where(red >= vals[:, j], red, vals[:, j]).astype(dt)
    else:
        red = np.zeros(n_o, dtype=dt)
        with np.errstate(all="ignore"):
            for j in range(n_r):
                red = (red.astype(np.uint64) + vals[:, j].astype(np.uint64)).astype(np.int64) if dt == np.int64 else (red + vals[:, j]).astype(dt)
    if a.mode == 3 and a.split == 1:  # chunk-wise staged: per-chunk partials
        chunk = 32 * 2 * (16 // np.dtype(dt).itemsize) * STAGED_U
        nch = (n_r + chunk - 1) // chunk
        part = np.zeros((n_o, nch), dtype=dt)
        for c in range(nch):
            sub = vals[:, c * chunk:(c + 1) * chunk]
            acc2 = np.full(n_o, -np.inf, dtype=dt) if a.red_kind == 2 else np.zeros(n_o, dtype=dt)
            for j in range(sub.shape[1]):
                acc2 = (np.where(acc2 >= sub[:, j], acc2, sub[:, j]) if a.red_kind == 2 else acc2 + sub[:, j]).astype(dt)
            part[:, c] = acc2
        mem.view(a.red_out.ref, dt)[: n_o * nch] = part.reshape(-1)
        return
    oo = np.arange(n_o, dtype=np.int64)
    mem.view(a.red_out.ref, dt)[leaf_offsets(a.red_out, oo, np.zeros_like(oo))] = red


def run_dot(mem, a, dt):
    A, B, Cm = mem.view(a.a, dt), mem.view(a.b, dt), mem.view(a.c, dt)
    i = np.arange(a.m)[:, None]
    j = np.arange(a.n)[None, :]
    acc = np.zeros((a.m, a.n), dtype=dt)
    for k in range(a.k):
        acc = (acc + (A[i * a.a_sm + k * a.a_sk] * B[k * a.b_sk + j * a.b_sn]).astype(dt)).astype(dt)
    Cm[i * a.c_sm + j * a.c_sn] = acc


def _gather4(buf, shape, strides):
    idx = np.zeros(shape, dtype=np.int64)
    for ax in range(4):
        sh = [1, 1, 1, 1]
        sh[ax] = shape[ax]
        idx = idx + np.arange(shape[ax]).reshape(sh) * strides[ax]
    return buf[idx], idx


def run_conv(mem, a, dt):
    from oracle import interp

    X, Y, O = mem.view(a.x, dt), mem.view(a.y, dt), mem.view(a.out, dt)
    et = 0 if dt == np.float32 else 1
    L = interp.lib()

    def p(arr):
        return arr.ctypes.data_as(interp.ctypes.c_void_p)

    if a.op in (3, 4):  # MaxPool / MaxPoolBackprop (IR extension)
        x, _ = np.ascontiguousarray(_gather4(X, (a.N, a.C, a.H, a.W), a.xs)[0]), None
        if a.op == 3:
            oshape = (a.N, a.C, a.Ho, a.Wo)
            out = np.empty(oshape, dtype=dt)
            L.orc_maxpool(et, p(x), p(out), a.N, a.C, a.H, a.W, a.R, a.S, a.sh, a.sw, a.pt, a.pl, a.Ho, a.Wo)
        else:
            d = np.ascontiguousarray(_gather4(Y, (a.N, a.C, a.Ho, a.Wo), a.ys)[0])
            oshape = (a.N, a.C, a.H, a.W)
            out = np.empty(oshape, dtype=dt)
            L.orc_maxpool_bwd(et, p(x), p(d), p(out), a.N, a.C, a.H, a.W, a.R, a.S, a.sh, a.sw, a.pt, a.pl, a.Ho, a.Wo)
    elif a.op == 0:
        x, _ = _gather4(X, (a.N, a.C, a.H, a.W), a.xs)
        f, _ = _gather4(Y, (a.K, a.C, a.R, a.S), a.ys)
        oshape = (a.N, a.K, a.Ho, a.Wo)
        out = np.empty(oshape, dtype=dt)
        x, f = np.ascontiguousarray(x), np.ascontiguousarray(f)
        L.orc_conv2d(et, p(x), p(f), p(out), a.N, a.C, a.H, a.W, a.K, a.R, a.S, a.sh, a.sw, a.pt, a.pl, a.Ho, a.Wo)
    elif a.op == 1:
        d, _ = _gather4(X, (a.N, a.K, a.Ho, a.Wo), a.xs)
        f, _ = _gather4(Y, (a.K, a.C, a.R, a.S), a.ys)
        oshape = (a.N, a.C, a.H, a.W)
        out = np.empty(oshape, dtype=dt)
        d, f = np.ascontiguousarray(d), np.ascontiguousarray(f)
        L.orc_conv_bwd_data(et, p(d), p(f), p(out), a.N, a.C, a.H, a.W, a.K, a.R, a.S, a.Ho, a.Wo, a.pt, a.pl, a.sh, a.sw)
    else:
        x, _ = _gather4(X, (a.N, a.C, a.H, a.W), a.xs)
        d, _ = _gather4(Y, (a.N, a.K, a.Ho, a.Wo), a.ys)
        oshape = (a.K, a.C, a.R, a.S)
        out = np.empty(oshape, dtype=dt)
        x, d = np.ascontiguousarray(x), np.ascontiguousarray(d)
        L.orc_conv_bwd_filter(et, p(x), p(d), p(out), a.N, a.C, a.H, a.W, a.K, a.R, a.S, a.Ho, a.Wo, a.pt, a.pl, a.sh, a.sw)
    _, idx = _gather4(O, oshape, a.os)
    O[idx] = out


def _rna_tf32(x: np.ndarray) -> np.ndarray:
    """cvt.rna.tf32.f32: round to nearest (ties away) keeping 10 mantissa bits."""
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    fin = np.isfinite(x)
    r = ((b + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return np.where(fin, r.view(np.float32), x.astype(np.float32))


def _gather_offsets(a, r, k):
    g, st = list(a.geo), list(a.st)
    valid = np.ones(np.broadcast(r, k).shape, dtype=bool)
    if a.mode == 1:
        HoWo, RS = g[6] * g[7], g[4] * g[5]
        n, pq = r // HoWo, r % HoWo
        pp, q = pq // g[7], pq % g[7]
        c, rs = k // RS, k % RS
        rr, ss = rs // g[5], rs % g[5]
        h, w = pp * g[8] - g[10] + rr, q * g[9] - g[11] + ss
        valid = (h >= 0) & (h < g[2]) & (w >= 0) & (w < g[3])
        off = n * st[0] + c * st[1] + h * st[2] + w * st[3]
    elif a.mode == 2:
        HW, RS = g[2] * g[3], g[4] * g[5]
        n, hw = r // HW, r % HW
        h, w = hw // g[3], hw % g[3]
        kk, rs = k // RS, k % RS
        rr, ss = rs // g[5], rs % g[5]
        pp, q = h + g[10] - rr, w + g[11] - ss
        valid = (pp >= 0) & (pp < g[6]) & (q >= 0) & (q < g[7])
        off = n * st[0] + kk * st[1] + pp * st[2] + q * st[3]
    elif a.mode == 3:
        d2, d01 = k % g[14], k // g[14]
        d1, d0 = d01 % g[13], d01 // g[13]
        off = r * a.s_r + d0 * st[0] + d1 * st[1] + d2 * st[2]
    elif a.mode == 4:
        RS, HoWo = g[4] * g[5], g[6] * g[7]
        c, rs = r // RS, r % RS
        rr, ss = rs // g[5], rs % g[5]
        n, pq = k // HoWo, k % HoWo
        pp, q = pq // g[7], pq % g[7]
        h, w = pp + rr - g[10], q + ss - g[11]
        valid = (h >= 0) & (h < g[2]) & (w >= 0) & (w < g[3])
        off = n * st[0] + c * st[1] + h * st[2] + w * st[3]
    else:  # 0 plain, 5 streaming (row-contiguous), 6 transposing (column-contiguous)
        off = r * a.s_r + k * a.s_k
    return np.where(valid, off, -1)


def run_split(mem, a):
    src = mem.view(a.src, np.float32)
    if a.mode == 7:  # lo plane only: the source is the hi operand (the MMA truncates it)
        x = src[: a.rows * a.kp].copy()
        hi = (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
        mem.view(a.lo, np.float32)[: a.rows * a.kp] = (x - hi).astype(np.float32)
        return
    r = np.arange(a.rows, dtype=np.int64)[:, None]
    k = np.arange(a.kp, dtype=np.int64)[None, :]
    off = _gather_offsets(a, r, np.minimum(k, max(a.k - 1, 0)))
    ok = (k < a.k) & (off >= 0)
    x = np.where(ok, src[np.clip(off, 0, src.size - 1)], 0.0).astype(np.float32)
    hi = _rna_tf32(x)
    lo = _rna_tf32((x - hi).astype(np.float32))
    mem.view(a.hi, np.float32)[: a.rows * a.kp] = hi.reshape(-1)
    mem.view(a.lo, np.float32)[: a.rows * a.kp] = lo.reshape(-1)


def _tf32(x):
    """What kind::tf32 reads of an fp32 operand: its top 19 bits (truncation)."""
    return (np.ascontiguousarray(x).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)


def _plane(mem, ref, rows, kp, k, ld_mn):
    """[rows, kp] operand: a K-major plane, or an MN-major tensor (element
    (r, k) at k * ld_mn + r, columns past K zero)."""
    v = mem.view(ref, np.float32)
    if ld_mn > 0:
        out = np.zeros((rows, kp), dtype=np.float32)
        out[:, :k] = v[np.arange(k)[None, :] * ld_mn + np.arange(rows)[:, None]]
        return _tf32(out)
    return _tf32(v[: rows * kp].reshape(rows, kp))


def run_tc(mem, a):
    A = (_plane(mem, a.a_hi, a.M, a.kp_a, a.K, a.a_ld_mn), _plane(mem, a.a_lo, a.M, a.kp_a, a.K, a.a_ld_mn))
    B = (_plane(mem, a.b_hi, a.N, a.kp_b, a.K, a.b_ld_mn), _plane(mem, a.b_lo, a.N, a.kp_b, a.K, a.b_ld_mn))
    splits = max(1, a.k_splits)
    i = np.arange(a.M, dtype=np.int64)[:, None]
    j = np.arange(a.N, dtype=np.int64)[None, :]
    C = mem.view(a.c, np.float32)
    for z in range(splits):
        k0 = z * a.k_per_split if splits > 1 else 0
        k1 = min(a.K, k0 + a.k_per_split) if splits > 1 else a.K
        sl = slice(k0, k1)
        c = (A[0][:, sl] @ B[0][:, sl].T + A[0][:, sl] @ B[1][:, sl].T + A[1][:, sl] @ B[0][:, sl].T).astype(np.float32)
        base = z * a.split_stride if splits > 1 else 0
        if a.epi_kind:  # fused epilogue (gfb200.h gfb_tc_args): dense [M, N] operands, pitch N
            with np.errstate(all="ignore"):
                if a.epi_kind == 1:
                    c = (c + mem.view(a.e_bias, np.float32)[: a.N][None, :]).astype(np.float32)
                    y = np.where(c > 0, c, np.float32(0)).astype(np.float32)
                    mem.view(a.e_out2, np.float32)[: a.M * a.N] = y.reshape(-1)
                else:  # the Relu-gradient mask, evaluated the graph's way: Maximum(Relu(x) / x, 0)
                    x = mem.view(a.e_aux2, np.float32)[: a.M * a.N].reshape(a.M, a.N)
                    r = (np.where(x > 0, x, np.float32(0)) / x).astype(np.float32)
                    c = (c * np.where(r >= 0, r, np.float32(0))).astype(np.float32)
                    y = c
                if a.epi_flags & 2:
                    hi = (np.ascontiguousarray(y).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
                    mem.view(a.e_lo, np.float32)[: a.M * a.N] = (y - hi).astype(np.float32).reshape(-1)
        if a.c_rdiv > 0:
            off = (i // a.c_rdiv) * a.c_s_hi + (i % a.c_rdiv) * a.c_s_lo + j * a.c_sn
        else:
            off = i * a.c_sm + j * a.c_sn
        C[base + off] = c


def _f16_scale(mx):
    """gemm_f16.cu / tc_prims.cuh f16_tile_scale: 2^(14 - floor(log2 mx))."""
    if not (mx > 0) or not np.isfinite(mx):
        return np.float32(1.0)
    e = int(np.frexp(np.float32(mx))[1])
    return np.float32(2.0 ** min(15 - e, 126))


def _f16_split(y, R, Cc):
    """fp16 hi / lo planes and the 128 x 128 tile scale grid of y [R, Cc]."""
    tr, tc = (R + 127) // 128, (Cc + 127) // 128
    sc = np.ones((tr, tc), dtype=np.float32)
    full = np.empty((R, Cc), dtype=np.float32)
    with np.errstate(all="ignore"):
        for i in range(tr):
            for j in range(tc):
                blk = y[128 * i:128 * (i + 1), 128 * j:128 * (j + 1)]
                fin = np.abs(blk)[np.isfinite(blk)]  # the scale counts finite values only
                sc[i, j] = _f16_scale(fin.max() if fin.size else 0.0)
                full[128 * i:128 * (i + 1), 128 * j:128 * (j + 1)] = sc[i, j]
        v = (y * full).astype(np.float32)
        hi = v.astype(np.float16)
        lo = (v - hi.astype(np.float32)).astype(np.float16)
    return hi, lo, sc


def run_split16(mem, a):
    src = mem.view(a.src, np.float32)
    y = src[np.arange(a.rows)[:, None] * a.ld + np.arange(a.cols)[None, :]]
    hi, lo, sc = _f16_split(y, a.rows, a.cols)
    mem.view(a.hi, np.float16)[: a.rows * a.cols] = hi.reshape(-1)
    mem.view(a.lo, np.float16)[: a.rows * a.cols] = lo.reshape(-1)
    mem.view(a.sc, np.float32)[: sc.size] = sc.reshape(-1)


def _plane16(mem, ref, scref, rows, kp, k, ld_mn, sc_r, sc_k):
    """[rows, k] operand of the fp16 GEMM, unscaled (exact in float64)."""
    v = mem.view(ref, np.float16)
    r = np.arange(rows)[:, None]
    kk = np.arange(k)[None, :]
    x = v[kk * ld_mn + r] if ld_mn > 0 else v[r * kp + kk]
    s = mem.view(scref, np.float32)[(r // 128) * sc_r + (kk // 128) * sc_k]
    return x.astype(np.float64) / s.astype(np.float64)


def run_f16p(mem, a):
    """gfb_gemm_f16p_kernel: sum over 128-K chunks of (Ahi Bhi + Ahi Blo +
    Alo Bhi) / (s_a s_b), then the fused epilogue (fp32 elementwise ops as
    in run_tc, fp16 planes of y when epi_flags bit 2 is set)."""
    Ah = _plane16(mem, a.a_hi, a.a_sc, a.M, a.kp_a, a.K, a.a_ld_mn, a.a_sc_r, a.a_sc_k)
    Al = _plane16(mem, a.a_lo, a.a_sc, a.M, a.kp_a, a.K, a.a_ld_mn, a.a_sc_r, a.a_sc_k)
    Bh = _plane16(mem, a.b_hi, a.b_sc, a.N, a.kp_b, a.K, a.b_ld_mn, a.b_sc_r, a.b_sc_k)
    Bl = _plane16(mem, a.b_lo, a.b_sc, a.N, a.kp_b, a.K, a.b_ld_mn, a.b_sc_r, a.b_sc_k)
    splits = max(1, a.k_splits)
    i = np.arange(a.M, dtype=np.int64)[:, None]
    j = np.arange(a.N, dtype=np.int64)[None, :]
    C = mem.view(a.c, np.float32)
    for z in range(splits):
        k0 = z * a.k_per_split if splits > 1 else 0
        k1 = min(a.K, k0 + a.k_per_split) if splits > 1 else a.K
        sl = slice(k0, k1)
        c = (Ah[:, sl] @ Bh[:, sl].T + Ah[:, sl] @ Bl[:, sl].T + Al[:, sl] @ Bh[:, sl].T).astype(np.float32)
        base = z * a.split_stride if splits > 1 else 0
        if a.epi_kind or a.epi_flags & 4:
            y = c
            with np.errstate(all="ignore"):
                if a.epi_kind == 1:
                    c = (c + mem.view(a.e_bias, np.float32)[: a.N][None, :]).astype(np.float32)
                    y = np.where(c > 0, c, np.float32(0)).astype(np.float32)
                    if a.epi_flags & 1:
                        mem.view(a.e_out2, np.float32)[: a.M * a.N] = y.reshape(-1)
                    if a.epi_flags & 8:  # mask bytes of x = c: 1 -> 1.0, 2 -> -0.0, 0 -> +0.0
                        code = np.where((c > 0) & (c < np.inf), 1, np.where(c < 0, 2, 0)).astype(np.uint8)
                        mem.view(a.e_mask, np.uint8)[: a.M * a.N] = code.reshape(-1)
                elif a.epi_kind == 2:
                    if a.epi_flags & 16:
                        code = mem.view(a.e_mask, np.uint8)[: a.M * a.N].reshape(a.M, a.N)
                        r = np.where(code == 1, np.float32(1), np.where(code == 2, np.float32(-0.0), np.float32(0)))
                        c = (c * r.astype(np.float32)).astype(np.float32)
                    else:
                        x = mem.view(a.e_aux2, np.float32)[: a.M * a.N].reshape(a.M, a.N)
                        r = (np.where(x > 0, x, np.float32(0)) / x).astype(np.float32)
                        c = (c * np.where(r >= 0, r, np.float32(0))).astype(np.float32)
                    y = c
            if a.epi_flags & 4:
                hi, lo, sc = _f16_split(y, a.M, a.N)
                mem.view(a.e_hi, np.float16)[: a.M * a.N] = hi.reshape(-1)
                mem.view(a.e_lo, np.float16)[: a.M * a.N] = lo.reshape(-1)
                mem.view(a.e_sc, np.float32)[: sc.size] = sc.reshape(-1)
        if a.epi_flags & 64:  # 32-row column partials: each lane's 8 rows in order, then (p0 + p1) + (p2 + p3)
            rp = (a.M + 31) // 32
            yy = np.zeros((rp * 32, a.N), dtype=np.float32)
            yy[: a.M] = y
            g = yy.reshape(rp, 8, 4, a.N)  # row 32 b + 4 i + g
            part = np.zeros((rp, 4, a.N), dtype=np.float32)
            for ii in range(8):
                part = (part + g[:, ii]).astype(np.float32)
            tot = ((part[:, 0] + part[:, 1]).astype(np.float32) + (part[:, 2] + part[:, 3]).astype(np.float32)).astype(np.float32)
            mem.view(a.e_csum, np.float32)[: rp * a.N] = tot.reshape(-1)
        if not a.epi_flags & 32:
            C[base + i * a.c_sm + j * a.c_sn] = c


def _trunc_split(x):
    """The converter warps' split (gemm_tc.cu split_rows): hi = x with the 13
    low mantissa bits cleared, lo = x - hi rounded to the TF32 the MMA reads."""
    hi = (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    lo = (x - hi).astype(np.float32)
    return hi, (lo.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def run_tcg(mem, a):
    """gfb_conv_tcg_kernel: gather A rows (n, y, x) x k = (r, s, c) from the
    channel-contiguous activation, split it like the kernel, contract with
    the B planes."""
    src = mem.view(a.a, np.float32)
    M, K, C = a.M, a.K, (a.C or 32 * a.CB)
    row = np.arange(M, dtype=np.int64)
    n, rem = row // (a.Y * a.X), row % (a.Y * a.X)
    h0 = (rem // a.X) * a.sy + a.oy
    w0 = (rem % a.X) * a.sx + a.ox
    k = np.arange(K, dtype=np.int64)
    c, rs = k % C, k // C
    dh, dw = a.ksign * (rs // a.S), a.ksign * (rs % a.S)
    h = h0[:, None] + dh[None, :]
    w = w0[:, None] + dw[None, :]
    ok = (h >= 0) & (h < a.H) & (w >= 0) & (w < a.W)
    off = n[:, None] * a.xs0 + h * a.xs2 + w * a.xs3 + c[None, :]
    x = np.where(ok, src[np.where(ok, off, 0)], np.float32(0)).astype(np.float32)
    ahi, alo = _trunc_split(x)
    bhi = mem.view(a.b_hi, np.float32)[: a.N * K].reshape(a.N, K).astype(np.float64)
    blo = mem.view(a.b_lo, np.float32)[: a.N * K].reshape(a.N, K).astype(np.float64)
    ahi, alo = ahi.astype(np.float64), alo.astype(np.float64)
    out = (ahi @ bhi.T + ahi @ blo.T + alo @ bhi.T).astype(np.float32)
    i = row[:, None]
    j = np.arange(a.N, dtype=np.int64)[None, :]
    mem.view(a.c, np.float32)[(i // a.c_rdiv) * a.c_s_hi + (i % a.c_rdiv) * a.c_s_lo + j * a.c_sn] = out


def run_stem(mem, a):
    """gfb_conv_stem_kernel: rows (n, y, x), k = (r, s, c) over (R, S, C) reads
    x[n, c, y + oy + r, x + ox + s] through strides (xs0, pad[0], xs2, xs3),
    zero outside; output row (n, y, x) at n*c_s_hi + y*c_sm + x*c_s_lo."""
    src = mem.view(a.a, np.float32)
    M, K, C = a.M, a.K, a.C
    R = K // (C * a.S)
    row = np.arange(M, dtype=np.int64)
    n, rem = row // (a.Y * a.X), row % (a.Y * a.X)
    y, x = rem // a.X, rem % a.X
    k = np.arange(K, dtype=np.int64)
    c, tap = k % C, k // C
    r, s = tap // a.S, tap % a.S
    h = (y + a.oy)[:, None] + r[None, :]
    w = (x + a.ox)[:, None] + s[None, :]
    ok = (h >= 0) & (h < a.H) & (w >= 0) & (w < a.W)
    off = n[:, None] * a.xs0 + c[None, :] * a.pad[0] + h * a.xs2 + w * a.xs3
    xv = np.where(ok, src[np.where(ok, off, 0)], np.float32(0)).astype(np.float32)
    ahi, alo = (v.astype(np.float64) for v in _trunc_split(xv))
    kp = a.pad[1]
    bhi = mem.view(a.b_hi, np.float32)[: a.N * kp].reshape(a.N, kp)[:, :K].astype(np.float64)
    blo = mem.view(a.b_lo, np.float32)[: a.N * kp].reshape(a.N, kp)[:, :K].astype(np.float64)
    out = (ahi @ bhi.T + ahi @ blo.T + alo @ bhi.T).astype(np.float32)
    j = np.arange(a.N, dtype=np.int64)[None, :]
    mem.view(a.c, np.float32)[(n * a.c_s_hi + y * a.c_sm + x * a.c_s_lo)[:, None] + j * a.c_sn] = out


def run_stemh(mem, a):
    """gfb_conv_stemh_kernel: the stem's gather in 2xFP16 -- one activation
    scale per 4 x 32 output tile (the largest finite |x| of its input patch,
    all channels), one filter scale per output channel; products in float64,
    rounded to fp32, then (/ u) / t_n."""
    src = mem.view(a.a, np.float32)
    M, K, C = a.M, a.K, a.C
    R = K // (C * a.S)
    row = np.arange(M, dtype=np.int64)
    n, rem = row // (a.Y * a.X), row % (a.Y * a.X)
    y, x = rem // a.X, rem % a.X
    k = np.arange(K, dtype=np.int64)
    c, tap = k % C, k // C
    r, s = tap // a.S, tap % a.S
    h = (y + a.oy)[:, None] + r[None, :]
    w = (x + a.ox)[:, None] + s[None, :]
    ok = (h >= 0) & (h < a.H) & (w >= 0) & (w < a.W)
    off = n[:, None] * a.xs0 + c[None, :] * a.xs1 + h * a.xs2 + w * a.xs3
    xv = np.where(ok, src[np.where(ok, off, 0)], np.float32(0)).astype(np.float32)
    # tile scales: the patch of tile (n, ty, tx) spans rows ty*4 + oy .. + 4 + R - 2
    # and columns tx*32 + ox .. + 32 + S - 2 (clipped to the image), all channels
    tile = (n * ((a.Y + 3) // 4) + y // 4) * ((a.X + 31) // 32) + x // 32
    u = np.ones(int(tile.max()) + 1 if M else 0, dtype=np.float32)
    xa = np.zeros((a.H, a.W), dtype=np.float64)
    for t in np.unique(tile):
        i = int(np.nonzero(tile == t)[0][0])
        y0, x0 = (y[i] // 4) * 4 + a.oy, (x[i] // 32) * 32 + a.ox
        hh = np.arange(max(0, y0), min(a.H, y0 + 4 + R - 1), dtype=np.int64)
        ww = np.arange(max(0, x0), min(a.W, x0 + 32 + a.S - 1), dtype=np.int64)
        cc = np.arange(C, dtype=np.int64)
        if hh.size and ww.size:
            pv = src[n[i] * a.xs0 + cc[:, None, None] * a.xs1 + hh[None, :, None] * a.xs2 + ww[None, None, :] * a.xs3]
            fin = np.abs(pv)[np.isfinite(pv)]
            u[t] = _f16_scale(fin.max() if fin.size else 0.0)
    with np.errstate(all="ignore"):
        v = (xv * u[tile][:, None]).astype(np.float32)
        ahi = v.astype(np.float16)
        alo = (v - ahi.astype(np.float32)).astype(np.float16)
        wt = mem.view(a.w, np.float32)
        j = np.arange(a.N, dtype=np.int64)
        wv = wt[j[:, None] * a.ws0 + c[None, :] * a.ws1 + r[None, :] * a.ws2 + s[None, :] * a.ws3].astype(np.float32)
        t_n = np.array([_f16_scale((lambda f: f.max() if f.size else 0.0)(np.abs(row_)[np.isfinite(row_)])) for row_ in wv],
                       dtype=np.float32)
        b = (wv * t_n[:, None]).astype(np.float32)
        bhi = b.astype(np.float16)
        blo = (b - bhi.astype(np.float32)).astype(np.float16)
        A = (ahi.astype(np.float64), alo.astype(np.float64))
        B = (bhi.astype(np.float64), blo.astype(np.float64))
        out = (A[0] @ B[0].T + A[0] @ B[1].T + A[1] @ B[0].T).astype(np.float32)
        out = ((out * (np.float32(1) / u[tile])[:, None]).astype(np.float32) * (np.float32(1) / t_n)[None, :]).astype(np.float32)
    mem.view(a.c, np.float32)[(n * a.c_s_hi + y * a.c_sm + x * a.c_s_lo)[:, None] + j[None, :] * a.c_sn] = out
    if a.flags & 1:  # the Relu side output (x > 0 ? x : 0)
        mem.view(a.c2, np.float32)[(n * a.c_s_hi + y * a.c_sm + x * a.c_s_lo)[:, None] + j[None, :] * a.c_sn] = \
            np.where(out > 0, out, np.float32(0)).astype(np.float32)


def run_stemwh(mem, a, grid):
    """gfb_conv_stemwh_kernel: CTA z's partial dW[k, n] over its contiguous
    range of 2 x 32 output-pixel tiles (float64 sums, rounded to fp32; the
    kernel's per-tile 2xFP16 scaling is exact to ~2^-22 and not modelled)."""
    src, dy = mem.view(a.a, np.float32), mem.view(a.w, np.float32)
    K, C, S = a.K, a.C, a.S
    R = K // (C * S)
    tiles_x, tiles_y = (a.X + 31) // 32, (a.Y + 1) // 2
    nimg = a.M // (a.Y * a.X)
    ntiles = nimg * tiles_y * tiles_x
    per = (ntiles + grid - 1) // grid
    k = np.arange(K, dtype=np.int64)
    c, tap = k % C, k // C
    r, s = tap // S, tap % S
    part = mem.view(a.c, np.float32)
    for z in range(grid):
        acc = np.zeros((K, a.N))
        for it in range(min(ntiles, z * per), min(ntiles, (z + 1) * per)):
            tx, rr = it % tiles_x, it // tiles_x
            ty, n = rr % tiles_y, rr // tiles_y
            yy, xx = np.meshgrid(np.arange(ty * 2, min(a.Y, ty * 2 + 2)), np.arange(tx * 32, min(a.X, tx * 32 + 32)), indexing="ij")
            yy, xx = yy.reshape(-1).astype(np.int64), xx.reshape(-1).astype(np.int64)
            d = dy[n * a.ws0 + yy[:, None] * a.ws2 + xx[:, None] * a.ws3 + np.arange(a.N)[None, :] * a.ws1].astype(np.float64)
            h = (yy + a.oy)[:, None] + r[None, :]
            w = (xx + a.ox)[:, None] + s[None, :]
            ok = (h >= 0) & (h < a.H) & (w >= 0) & (w < a.W)
            off = n * a.xs0 + c[None, :] * a.xs1 + h * a.xs2 + w * a.xs3
            xv = np.where(ok, src[np.where(ok, off, 0)], 0.0).astype(np.float64)
            acc += xv.T @ d
        part[z * K * a.N:(z + 1) * K * a.N] = acc.astype(np.float32).reshape(-1)


def run_tcx(mem, a):
    """gfb_conv_tcx_kernel: rows are output pixels (n, y, x); the TMA box for
    K-block (r, s, cb) reads act[n, y*sy + oy + ksign*r, x*sx + ox + ksign*s,
    c] (zero outside the tensor)."""
    src = mem.view(a.a, np.float32)
    Cc, Wd, Hd, Nd = list(a.a_dims)
    sc, sw, sh, sn = list(a.a_strides)
    K = a.K
    n, y, x = np.meshgrid(np.arange(a.No), np.arange(a.Yo), np.arange(a.Xo), indexing="ij")
    n, y, x = (v.reshape(-1, 1).astype(np.int64) for v in (n, y, x))
    k = np.arange(K, dtype=np.int64)[None, :]
    C = 32 * a.CB
    c, rs = k % C, k // C
    h = y * a.sy + a.oy + a.ksign * (rs // a.S)
    w = x * a.sx + a.ox + a.ksign * (rs % a.S)
    ok = (h >= 0) & (h < Hd) & (w >= 0) & (w < Wd)
    off = n * sn + h * sh + w * sw + c * sc
    v = np.where(ok, src[np.where(ok, off, 0)], np.float32(0)).astype(np.float32)
    ahi, alo = _trunc_split(v)
    bhi = mem.view(a.b_hi, np.float32)[: a.N * K].reshape(a.N, K).astype(np.float64)
    blo = mem.view(a.b_lo, np.float32)[: a.N * K].reshape(a.N, K).astype(np.float64)
    ahi, alo = ahi.astype(np.float64), alo.astype(np.float64)
    out = (ahi @ bhi.T + ahi @ blo.T + alo @ bhi.T).astype(np.float32)
    j = np.arange(a.N, dtype=np.int64)[None, :]
    mem.view(a.c, np.float32)[n * a.o_n + y * a.o_y + x * a.o_x + j * a.c_sn] = out


def _ch_scale_vec(m):
    return np.array([_f16_scale(v) for v in m], dtype=np.float32)


def run_chmax(mem, a):
    x = mem.view(a.src, np.float32)[: a.P * a.C].reshape(a.P, a.C)
    part = mem.view(a.partial, np.float32)
    ax = np.where(np.isfinite(x), np.abs(x), 0)
    part[: a.C] = np.maximum(part[: a.C], ax.max(axis=0))


def run_chsplit(mem, a):
    s = _ch_scale_vec(mem.view(a.partial, np.float32)[: a.C])
    mem.view(a.sc, np.float32)[: a.C] = s
    x = mem.view(a.src, np.float32)[: a.P * a.C].reshape(a.P, a.C)
    with np.errstate(all="ignore"):
        v = (x * s[None, :]).astype(np.float32)
        hi = v.astype(np.float16)
        lo = (v - hi.astype(np.float32)).astype(np.float16)
    mem.view(a.hi, np.float16)[: a.P * a.C] = hi.reshape(-1)
    mem.view(a.lo, np.float16)[: a.P * a.C] = lo.reshape(-1)


def run_fsplit(mem, a):
    w = mem.view(a.w, np.float32)
    sc = mem.view(a.sc, np.float32)
    k = np.arange(a.K, dtype=np.int64)
    d2, d01 = k % a.e2, k // a.e2
    d1, d0 = d01 % a.e1, d01 // a.e1
    rows = np.arange(a.rows, dtype=np.int64)[:, None]
    b = (w[rows * a.s_r + (d0 * a.t0 + d1 * a.t1 + d2 * a.t2)[None, :]] / sc[d2][None, :]).astype(np.float32)
    t = _ch_scale_vec(np.where(np.isfinite(b), np.abs(b), 0).max(axis=1))
    v = (b * t[:, None]).astype(np.float32)
    hi = v.astype(np.float16)
    lo = (v - hi.astype(np.float32)).astype(np.float16)
    mem.view(a.hi, np.float16)[: a.rows * a.K] = hi.reshape(-1)
    mem.view(a.lo, np.float16)[: a.rows * a.K] = lo.reshape(-1)
    mem.view(a.inv, np.float32)[: a.rows] = (1.0 / t).astype(np.float32)


def run_tcxh(mem, a):
    """gfb_conv_tcxh_kernel: the tcx gather over the fp16 activation planes
    (64-channel K-blocks), products in float64, then times 1 / t_n."""
    Cc, Wd, Hd, Nd = list(a.a_dims)
    sc, sw, sh, sn = list(a.a_strides)
    K = a.K
    n, y, x = np.meshgrid(np.arange(a.No), np.arange(a.Yo), np.arange(a.Xo), indexing="ij")
    n, y, x = (v.reshape(-1, 1).astype(np.int64) for v in (n, y, x))
    k = np.arange(K, dtype=np.int64)[None, :]
    C = 64 * a.CB
    c, rs = k % C, k // C
    h = y * a.sy + a.oy + a.ksign * (rs // a.S)
    w = x * a.sx + a.ox + a.ksign * (rs % a.S)
    ok = (h >= 0) & (h < Hd) & (w >= 0) & (w < Wd)
    off = np.where(ok, n * sn + h * sh + w * sw + c * sc, 0)
    ahi = np.where(ok, mem.view(a.a_hi, np.float16)[off].astype(np.float64), 0.0)
    alo = np.where(ok, mem.view(a.a_lo, np.float16)[off].astype(np.float64), 0.0)
    bhi = mem.view(a.b_hi, np.float16)[: a.N * K].reshape(a.N, K).astype(np.float64)
    blo = mem.view(a.b_lo, np.float16)[: a.N * K].reshape(a.N, K).astype(np.float64)
    out = (ahi @ bhi.T + ahi @ blo.T + alo @ bhi.T).astype(np.float32)
    inv = mem.view(a.b_inv, np.float32)[: a.N]
    out = (out * inv[None, :]).astype(np.float32)
    j = np.arange(a.N, dtype=np.int64)[None, :]
    mem.view(a.c, np.float32)[n * a.o_n + y * a.o_y + x * a.o_x + j * a.c_sn] = out


def run_tcgwh(mem, a):
    """gfb_conv_tcgwh_kernel: dW[(r, s, c), k] = sum over output pixels of the
    x planes at the tap-shifted pixel times the dy planes, unscaled."""
    Cc, Wd, Hd, Nd = list(a.a_dims)
    K_, Wo, Ho, _ = list(a.b_dims)
    xs = np.zeros((Nd, Hd + 2 * 8, Wd + 2 * 8, Cc))  # zero border for the taps (|shift| <= 8 here)
    sc_a = mem.view(a.a_sc, np.float32)[:Cc].astype(np.float64)
    sc_b = mem.view(a.b_sc, np.float32)[:K_].astype(np.float64)
    xhl = (mem.view(a.a_hi, np.float16)[: Nd * Hd * Wd * Cc].astype(np.float64),
           mem.view(a.a_lo, np.float16)[: Nd * Hd * Wd * Cc].astype(np.float64))
    dhl = (mem.view(a.b_hi, np.float16)[: Nd * Ho * Wo * K_].astype(np.float64).reshape(-1, K_),
           mem.view(a.b_lo, np.float16)[: Nd * Ho * Wo * K_].astype(np.float64).reshape(-1, K_))
    R = a.M // (Cc * a.S)
    rows = []
    for r in range(R):
        for s_ in range(a.S):
            dy_ = r - a.pt
            dx_ = s_ - a.pl
            parts = []
            for xv in xhl:
                xs[:] = 0
                xs[:, 8:8 + Hd, 8:8 + Wd, :] = xv.reshape(Nd, Hd, Wd, Cc)
                win = xs[:, 8 + dy_:8 + dy_ + Ho, 8 + dx_:8 + dx_ + Wo, :].reshape(-1, Cc)
                parts.append(win)
            g = parts[0].T @ dhl[0] + parts[0].T @ dhl[1] + parts[1].T @ dhl[0]
            rows.append(g)
    dw = np.concatenate(rows, axis=0) / sc_a[np.arange(a.M) % Cc][:, None] / sc_b[None, :]
    dw = dw.astype(np.float32)
    i = np.arange(a.M, dtype=np.int64)[:, None]
    j = np.arange(a.N, dtype=np.int64)[None, :]
    C = mem.view(a.c, np.float32)
    if a.k_splits > 1:  # the whole sum in split 0, zeros in the others (the reduce pass adds them)
        C[i * a.N + j] = dw
        for z in range(1, a.k_splits):
            C[z * a.split_stride + i * a.N + j] = 0.0
    else:
        C[(i // Cc) * a.c_s_hi + (i % Cc) * a.c_s_lo + j * a.c_sn] = dw


def run_tcgg(mem, a):
    """gfb_conv_tcgg_kernel: generic row / K decompositions (gfb_tcgg_args)."""
    src = mem.view(a.a, np.float32)
    row = np.arange(a.M, dtype=np.int64)
    e12 = a.E1 * a.E2
    i0, rem = row // e12, row % e12
    i1, i2 = rem // a.E2, rem % a.E2
    rowoff = i0 * a.ro0 + i1 * a.ro1 + i2 * a.ro2
    if a.pad0 == 1:
        hr, wr = i0 * a.hm + a.h0, i1 * a.wm + a.w0
    else:
        hr, wr = i1 * a.hm + a.h0, i2 * a.wm + a.w0
    k = np.arange(a.K, dtype=np.int64)
    ke12 = a.Ke1 * a.Ke2
    k0, kr = k // ke12, k % ke12
    k1, k2 = kr // a.Ke2, kr % a.Ke2
    koff = a.kbase + k0 * a.ko0 + k1 * a.ko1 + k2 * a.ko2
    h = hr[:, None] + (k1 * a.kh + a.dh0)[None, :]
    w = wr[:, None] + (k2 * a.kw + a.dw0)[None, :]
    ok = (h >= 0) & (h < a.H) & (w >= 0) & (w < a.W)
    off = rowoff[:, None] + koff[None, :]
    x = np.where(ok, src[np.where(ok, off, 0)], np.float32(0)).astype(np.float32)
    ahi, alo = _trunc_split(x)
    ahi, alo = ahi.astype(np.float64), alo.astype(np.float64)
    bhi = mem.view(a.b_hi, np.float32)[: a.N * a.kp_b].reshape(a.N, a.kp_b)[:, : a.K].astype(np.float64)
    blo = mem.view(a.b_lo, np.float32)[: a.N * a.kp_b].reshape(a.N, a.kp_b)[:, : a.K].astype(np.float64)
    C = mem.view(a.c, np.float32)
    i = row[:, None]
    j = np.arange(a.N, dtype=np.int64)[None, :]
    kblocks = (a.K + 31) // 32
    for z in range(max(1, a.k_splits)):
        b0 = z * a.kb_per_split if a.k_splits > 1 else 0
        b1 = min(kblocks, b0 + a.kb_per_split) if a.k_splits > 1 else kblocks
        sl = slice(32 * b0, min(a.K, 32 * b1))
        c = (ahi[:, sl] @ bhi[:, sl].T + ahi[:, sl] @ blo[:, sl].T + alo[:, sl] @ bhi[:, sl].T).astype(np.float32)
        base = z * a.split_stride if a.k_splits > 1 else 0
        if a.c_rdiv > 0:
            off = (i // a.c_rdiv) * a.c_s_hi + (i % a.c_rdiv) * a.c_s_lo + j * a.c_sn
        else:
            off = i * a.c_sm + j * a.c_sn
        C[base + off] = c


def run_tcgw(mem, a):
    """gfb_conv_tcgw_kernel: MN-major weight gradient over channel-last x and
    dy, both operands split to TF32 hi/lo in the kernel (gfb_tcgw_args)."""
    X = mem.view(a.a, np.float32)
    Y = mem.view(a.b, np.float32)
    row = np.arange(a.M, dtype=np.int64)
    e12 = a.E1 * a.E2
    i0, rem = row // e12, row % e12
    i1, i2 = rem // a.E2, rem % a.E2
    rowoff = i0 * a.ro0 + i1 * a.ro1 + i2 * a.ro2 + a.kbase
    hr, wr = i0 + a.h0, i1 + a.w0
    k = np.arange(a.K, dtype=np.int64)
    ke12 = a.Ke1 * a.Ke2
    k0, kr = k // ke12, k % ke12
    k1, k2 = kr // a.Ke2, kr % a.Ke2
    h = hr[:, None] + k1[None, :]
    w = wr[:, None] + k2[None, :]
    ok = (h >= 0) & (h < a.H) & (w >= 0) & (w < a.W)
    off = rowoff[:, None] + (k0 * a.ko0 + k1 * a.ko1 + k2 * a.ko2)[None, :]
    x = np.where(ok, X[np.where(ok, off, 0)], np.float32(0)).astype(np.float32)
    ahi, alo = (v.astype(np.float64) for v in _trunc_split(x))
    yoff = (k0 * a.yo0 + k1 * a.yo1 + k2 * a.yo2)[None, :] + np.arange(a.N, dtype=np.int64)[:, None]
    bhi, blo = (v.astype(np.float64) for v in _trunc_split(Y[yoff].astype(np.float32)))
    C = mem.view(a.c, np.float32)
    i = row[:, None]
    j = np.arange(a.N, dtype=np.int64)[None, :]
    kblocks = (a.K + 31) // 32
    for z in range(max(1, a.k_splits)):
        b0 = z * a.kb_per_split if a.k_splits > 1 else 0
        b1 = min(kblocks, b0 + a.kb_per_split) if a.k_splits > 1 else kblocks
        sl = slice(32 * b0, min(a.K, 32 * b1))
        c = (ahi[:, sl] @ bhi[:, sl].T + ahi[:, sl] @ blo[:, sl].T + alo[:, sl] @ bhi[:, sl].T).astype(np.float32)
        base = z * a.split_stride if a.k_splits > 1 else 0
        if a.c_rdiv > 0:
            o = (i // a.c_rdiv) * a.c_s_hi + (i % a.c_rdiv) * a.c_s_lo + j * a.c_sn
        else:
            o = i * a.c_sm + j * a.c_sn
        C[base + o] = c


STAGED_U = 2  # csrc/ew_vm.cu StagedCfg<T, 2>


def _run_launch(mem, L):
    dt = DT.get(L.kind)
    if L.kind in (abi.K_EW_F32, abi.K_EW_F64, abi.K_EW_I64, abi.K_EW_U8, abi.K_EWS_F32, abi.K_EWS_F64, abi.K_EW1_F32,
                  abi.K_EW1_F64):
        run_ew(mem, L.args, dt)
    elif L.kind in (abi.K_DOT_F32, abi.K_DOT_F64, abi.K_DOT_SM_F32, abi.K_DOT_SM_F64, abi.K_DOT_TH_F32, abi.K_DOT_TH_F64):
        run_dot(mem, L.args, dt)
    elif L.kind in (abi.K_CONV_F32, abi.K_CONV_F64):
        run_conv(mem, L.args, dt)
    elif L.kind == abi.K_SPLIT_TF32:
        run_split(mem, L.args)
    elif L.kind in (abi.K_DOT_TC32, abi.K_DOT_TC32W, abi.K_DOT_TC32P):
        run_tc(mem, L.args)
    elif L.kind == abi.K_SPLIT_F16:
        run_split16(mem, L.args)
    elif L.kind == abi.K_DOT_F16P:
        run_f16p(mem, L.args)
    elif L.kind == abi.K_MEMSET:
        mem.view(L.args.buf, np.uint8)[: L.args.bytes] = 0
    elif L.kind == abi.K_CHMAX:
        run_chmax(mem, L.args)
    elif L.kind == abi.K_CHSPLIT:
        run_chsplit(mem, L.args)
    elif L.kind == abi.K_FSPLIT:
        run_fsplit(mem, L.args)
    elif L.kind in (abi.K_CONV_TCXH64, abi.K_CONV_TCXH128):
        run_tcxh(mem, L.args)
    elif L.kind in (abi.K_CONV_TCGWH64, abi.K_CONV_TCGWH128):
        run_tcgwh(mem, L.args)
    elif L.kind in (abi.K_CONV_TCG64, abi.K_CONV_TCG128):
        run_tcg(mem, L.args)
    elif L.kind in (abi.K_CONV_TCX64, abi.K_CONV_TCX128):
        run_tcx(mem, L.args)
    elif L.kind == abi.K_CONV_STEM64:
        run_stem(mem, L.args)
    elif L.kind in (abi.K_CONV_STEMH, abi.K_CONV_STEMH_C3R7):
        run_stemh(mem, L.args)
    elif L.kind == abi.K_CONV_STEMWH_C3R7:
        run_stemwh(mem, L.args, L.grid[0])
    elif L.kind in (abi.K_CONV_TCGW64, abi.K_CONV_TCGW128):
        run_tcgw(mem, L.args)
    elif L.kind in (abi.K_CONV_TCGG64, abi.K_CONV_TCGG128):
        run_tcgg(mem, L.args)
    elif L.kind == abi.K_ROWJIT:
        run_row(mem, L)
    else:
        raise NotImplementedError(L.kind)


def run_row(mem, L):
    """A row-fused launch (paper_1801_08058_b200/rowfuse.py) in reference
    semantics: its value program over whole [R, C] arrays, row reductions
    folded sequentially along the row, cross-row reductions sequentially in
    row-major order.  The kernel's per-team partials are emulated as
    (that full fold, then fold identities), so the second pass reproduces
    the reference's single sequential fold exactly."""
    spec, a = L.row_spec, L.args
    dt = np.float32 if spec.dtype == "float" else np.float64
    R, C = spec.R, spec.C
    rows = np.arange(R, dtype=np.int64)[:, None]
    cols = np.arange(C, dtype=np.int64)[None, :]

    def fold_seq(kind, vals):  # vals [..., n]: fold along the last axis from the identity
        acc = np.full(vals.shape[:-1], -np.inf if kind == 2 else 0.0, dtype=dt)
        with np.errstate(all="ignore"):
            for j in range(vals.shape[-1]):
                v = vals[..., j]
                acc = (np.where(acc >= v, acc, v) if kind == 2 else acc + v).astype(dt)
        return acc

    v = []
    for cls, e in spec.values:
        op = e[0]
        if op == "imm":
            raw = np.array([e[1]], dtype=np.uint64)
            x = raw.astype(np.uint32).view(np.float32)[0] if dt == np.float32 else raw.view(np.float64)[0]
            v.append(dt(x))
        elif op == "loadu":
            v.append(mem.view(a.refs[e[1]], dt)[0])
        elif op == "load":
            v.append(mem.view(a.refs[e[1]], dt)[rows * e[2] + cols * e[3]].copy())
        elif op == "loadr":
            v.append(mem.view(a.refs[e[1]], dt)[np.arange(R) * e[2]].copy())
        elif op == "colv":
            v.append(np.broadcast_to(mem.view(a.refs[e[1]], dt)[np.arange(C) * e[2]], (R, C)).copy())
        elif op == "bcast":
            x = v[e[1]]
            v.append(np.broadcast_to(np.asarray(x)[:, None] if np.ndim(x) == 1 else x, (R, C) if cls == "full" else (R,)).astype(dt))
        elif op == "un":
            v.append(_un(e[1], np.asarray(v[e[2]], dtype=dt), dt))
        elif op == "bin":
            v.append(_bin(e[1], np.asarray(v[e[2]], dtype=dt), np.asarray(v[e[3]], dtype=dt), dt))
        elif op == "rred":
            v.append(fold_seq(e[1], v[e[2]]))
        elif op == "xred":
            v.append(fold_seq(e[1], np.asarray(v[e[2]]).reshape(1, -1))[0])
        else:
            raise ValueError(e)
    for k, ref, s0, s1 in spec.stores:
        x = v[k]
        if np.ndim(x) == 2:
            mem.view(a.refs[ref], dt)[rows * s0 + cols * s1] = x
        else:
            mem.view(a.refs[ref], dt)[np.arange(R) * s0] = x
    for k, kind, ref in spec.xrow:
        part = np.full(spec.n_teams, -np.inf if kind == 2 else 0.0, dtype=dt)
        part[0] = v[k]
        mem.view(a.refs[ref], dt)[: spec.n_teams] = part


def allreduce_view(mem, a):
    dt = np.float32 if a.dtype == 0 else np.float64
    return mem.view(a.buf, dt)[: a.count]


def execute_ranks(lowered, inputs_per_rank: list, out_specs: list, allreduce=None) -> list:
    """Lock-step execution of one data-parallel plan on several emulated ranks.

    `allreduce(list_of_arrays)` sums in place (default: rank-order fp sum);
    a torch.distributed-backed callable makes this a real multi-process run."""
    mems, outs = [], []
    for ins in inputs_per_rank:
        o = [np.zeros(max(c, 1), dtype=d) for d, c in out_specs]
        mems.append(Memory(lowered, [np.ascontiguousarray(x).reshape(-1) for x in ins], o))
        outs.append(o)
    for L in lowered.launches:
        if L.kind == abi.K_ALLREDUCE:
            views = [allreduce_view(m, L.args) for m in mems]
            if allreduce is not None:
                allreduce(views, L.args.op)
            else:
                total = views[0].copy()
                for v in views[1:]:
                    total = np.maximum(total, v) if L.args.op == 1 else total + v
                for v in views:
                    v[:] = total
            continue
        for m in mems:
            _run_launch(m, L)
    return [[o[:c] for o, (_, c) in zip(os, out_specs)] for os in outs]


def execute(lowered, inputs: list, out_specs: list) -> list:
    """inputs: storage-order numpy arrays; out_specs: (dtype, count)."""
    outputs = [np.zeros(max(c, 1), dtype=d) for d, c in out_specs]
    mem = Memory(lowered, [np.ascontiguousarray(x).reshape(-1) for x in inputs], outputs)
    for L in lowered.launches:
        _run_launch(mem, L)
    return [o[:c] for o, (_, c) in zip(outputs, out_specs)]
