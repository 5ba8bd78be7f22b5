"""Runtime specialisation of the fused elementwise VM kernel (NVRTC).

The generic `gfb_ew_kernel` (csrc/ew_vm.cu) interprets a launch's program and
index maps from its argument block: a jump-table dispatch per VM instruction
and per-leaf branches on map kind, digit count and vector class.  On the
heaviest launches of a training step (config D's pool-window gradients, for
example: 25 VM instructions over 11 leaves) that interpretation, not HBM,
bounds the kernel.

Every launch's structure is fixed when the graph is compiled; only the slot
table (`tab`: arena / inputs / outputs of this run) changes between runs.
So, like nGraph's GPU transformer, which emitted CUDA C for its fused
elementwise kernels and compiled it with NVRTC, this module generates one
kernel per launch with the same semantics as the generic one (csrc/ew_vm.cu):
the program becomes straight-line code over register vectors (the operand
stack disappears), every index map becomes literal multiply-shift digit
arithmetic, and each leaf's load / store is the one its vector class needs.
The element operations are the generic kernel's own (csrc/ew_ops.cuh:
`bin1`, `apply_unary`, `fold`), so results are bit-identical; the tests
check that.

Compiled cubins are cached on disk (key: source + options + kernel headers);
the cache only saves compile time.  `GFB_JIT=0` disables specialisation.
If NVRTC is missing or a generated kernel fails to compile, the launch keeps
the generic CUDA kernel and a RuntimeWarning says so (`GFB_JIT_STRICT=1`,
set by the test suite, raises instead).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import threading
from concurrent.futures import ThreadPoolExecutor

from . import abi

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
CUDA_INCLUDE = os.environ.get("GFB_CUDA_INCLUDE", "/usr/local/cuda/include")
HEADERS = [os.path.join(CSRC, "ew_ops.cuh"), os.path.join(CSRC, "gfb_common.cuh"), os.path.join(INCLUDE, "gfb200.h")]
F_LOADP, F_LOADM, F_PUSH, F_STORE, F_UN, F_DOT, F_BIN = 1, 5, 6, 7, 8, 14, 16  # csrc/ew_ops.cuh

# kind -> (element type, vector width, min blocks per SM) of the generic kernel it replaces
KINDS = {
    abi.K_EW_F32: ("float", 8, 4),
    abi.K_EW_F64: ("double", 4, 4),
    abi.K_EW1_F32: ("float", 1, 4),
    abi.K_EW1_F64: ("double", 1, 4),
    abi.K_EWS_F32: ("float", 8, 4),  # chunk-wise staged launches (mode 3, split 1) only
    abi.K_EWS_F64: ("double", 4, 4),
}
OPTIONS = ["-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo"]
ENTRY = b"gfb_jit_ew"
# launches moving fewer bytes than this stay on the generic kernel
MIN_BYTES = int(os.environ.get("GFB_JIT_MIN_BYTES", 0))

_lock = threading.Lock()
_nvrtc = None
_kernels: dict = {}  # cubin digest -> kernel handle (libraries stay loaded for the process)
_header_digest = None


_warned: set = set()


def _warn_once(msg: str):
    import warnings

    if msg not in _warned:
        _warned.add(msg)
        warnings.warn(msg, RuntimeWarning, stacklevel=3)


def enabled() -> bool:
    return os.environ.get("GFB_JIT", "1") != "0"


def _lib_nvrtc():
    global _nvrtc
    if _nvrtc is None:
        cands = ["libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"]
        try:
            import nvidia.cuda_nvrtc as m  # torch's bundled NVRTC

            cands.insert(1, os.path.join(list(m.__path__)[0], "lib", "libnvrtc.so.12"))
        except Exception:
            pass
        err = None
        for c in cands:
            try:
                L = C.CDLL(c)
                break
            except OSError as e:
                err = e
        else:
            raise RuntimeError(f"NVRTC not found: {err}")
        vp, sz = C.c_void_p, C.c_size_t
        L.nvrtcCreateProgram.argtypes = [C.POINTER(vp), C.c_char_p, C.c_char_p, C.c_int, vp, vp]
        L.nvrtcCompileProgram.argtypes = [vp, C.c_int, C.POINTER(C.c_char_p)]
        L.nvrtcGetProgramLogSize.argtypes = [vp, C.POINTER(sz)]
        L.nvrtcGetProgramLog.argtypes = [vp, C.c_char_p]
        L.nvrtcGetCUBINSize.argtypes = [vp, C.POINTER(sz)]
        L.nvrtcGetCUBIN.argtypes = [vp, C.c_char_p]
        L.nvrtcDestroyProgram.argtypes = [C.POINTER(vp)]
        _nvrtc = L
    return _nvrtc


def _c_init(v) -> str:
    """C brace initialiser of a ctypes value, in field order."""
    if isinstance(v, C.Structure):
        return "{" + ",".join(_c_init(getattr(v, f)) for f, *_ in v._fields_) + "}"
    if isinstance(v, C.Array):
        return "{" + ",".join(_c_init(x) for x in v) + "}"
    if v is None:
        return "nullptr"
    if isinstance(v, int):
        return f"{v}ull" if v > 0x7FFFFFFF else str(v)
    raise TypeError(f"cannot initialise from {type(v)}")


def _mode_ok(args) -> bool:
    """ROW (1), COL (2) and the chunk-wise staged mode (3 with split 1: few
    long rows cut into chunks, one partial per (row, chunk))."""
    return args.mode in (1, 2) or (args.mode == 3 and args.split == 1)


def generate(kind: int, args: "abi.EwArgs", block: int = 256):
    """(CUDA C of one launch's specialised kernel, its dynamic shared memory
    bytes), or None when the generic kernel keeps the launch."""
    if kind not in KINDS or not _mode_ok(args):
        return None
    g = _Gen(kind, args, block)
    src = g.emit()
    return src, g.smem


def generate_merged(members, block: int):
    """One kernel running several single-block launches in order, a block
    barrier between them (their global writes are then visible to the whole
    block, and every load is a plain coherent load, never the read-only
    path).  `members`: [(kind, args)].  Returns (source, smem) or None."""
    gens = []
    for kind, args in members:
        if kind not in KINDS or not _mode_ok(args):
            return None
        gens.append(_Gen(kind, args, block))
    src = _kernel_source(gens)
    return src, max(g.smem for g in gens)


def _kernel_source(gens) -> str:
    block = gens[0].block
    merged = len(gens) > 1
    L = ['#include "ew_ops.cuh"', "using namespace gfb;",
         "__device__ __forceinline__ uint32_t mod_of(uint32_t q, uint32_t mul, uint32_t sh, uint32_t m) {"
         " return q - fast_div(q, mul, sh) * m; }"]
    if merged:  # later members read what earlier ones wrote in this kernel: coherent loads only
        L += ["#define GFB_LD(p) (*(p))", "#define GFB_LOADV(p, x) loadV_plain<T, V>((p), (x))"]
    else:
        L += ["#define GFB_LD(p) __ldg(p)", "#define GFB_LOADV(p, x) loadV<T, V>((p), (x))"]
    bodies = [g.member(i) for i, g in enumerate(gens)]
    L += bodies
    L.append(f'extern "C" __global__ void __launch_bounds__({block}, {max(1, 1024 // block)}) '
             "gfb_jit_ew(const __grid_constant__ gfb_ew_args pa) {")
    L.append("extern __shared__ __align__(16) unsigned char dyn[];")
    for i in range(len(gens)):
        if i:
            L.append("__syncthreads();")
        L.append(f"m{i}::run(pa, dyn);")
    L.append("}")
    return "\n".join(L) + "\n"


def _u32(x: int) -> str:
    return f"{x & 0xFFFFFFFF}u"


class _Gen:
    """Straight-line code for one gfb_ew_args (semantics of csrc/ew_vm.cu:
    `Ctx::load` / `Ctx::store`, `vm_run`, and the ROW / COL loops of
    gfb_ew_kernel, with every structural value a literal)."""

    def __init__(self, kind, a, block):
        self.t, self.V, self.minb = KINDS[kind]
        if a.mode == 3:
            # the chunk-wise staged kernel hands each lane 16-byte pieces
            # (csrc/ew_vm.cu sidx): generate over 16-byte vectors so the
            # lane-to-element map, and with it the fold order, is the same
            self.V //= 2
        self.a, self.block = a, block
        self.nl = a.nleaves
        self.leaves = [a.leaves[k] for k in range(self.nl)]
        self.ops = []
        # leaves with equal digit lists share their offset expressions
        self.map_of, self.maps = {}, []
        for k, L in enumerate(self.leaves):
            if L.mode == 1:
                continue
            key = self._digits(L)
            if key not in self.maps:
                self.maps.append(key)
            self.map_of[k] = self.maps.index(key)
        self.stored = {((w >> 8) & 0xFF) for w in a.prog[:a.ninstr] if (w & 0xFF) == F_STORE}
        self.n = 0

    @staticmethod
    def _digits(L):
        return (L.rlin, tuple((d.div_mul & 0xFFFFFFFF, d.div_sh, d.mod, d.mod_mul & 0xFFFFFFFF, d.mod_sh, d.stride, d.src)
                              for d in L.dig[:L.ndig]))

    # ---- index maps ----------------------------------------------------
    @staticmethod
    def _expr(digits, o, r, src=None):
        terms = []
        for mul, sh, mod, mmul, msh, stride, dsrc in digits:
            if src is not None and dsrc != src:
                continue
            n = r if dsrc else o
            q = f"fast_div({n}, {_u32(mul)}, {sh}u)"
            if mod:
                q = f"mod_of({q}, {_u32(mmul)}, {msh}u, {mod}u)"
            terms.append(f"{q} * {_u32(stride)}")
        return " + ".join(terms) if terms else "0u"

    def _rpart(self, m, r):
        rlin, digits = self.maps[m]
        return f"({r}) * {_u32(rlin)}" if rlin >= 0 else self._expr(digits, "0u", r, src=1)

    def _full_off(self, k, o, r):
        return self._expr(self.maps[self.map_of[k]][1], o, r)

    def _tmp(self):
        self.n += 1
        return f"t{self.n}"

    def _elem(self, k, v):
        vaxis = self.a.mode in (1, 3)
        o = "o" if vaxis else f"o + {v}u"
        r = f"r + {v}u" if vaxis else "r"
        return self._full_off(k, o, r)

    # ---- loads / stores (Ctx::load / Ctx::store) ------------------------
    def load(self, k, full, out):
        L, V, T = self.leaves[k], self.V, "T"
        x = self._tmp()
        out.append(f"T {x}[V];")
        if L.mode == 1:
            out.append(f"{{ const T s = from_bits<T>({L.splat}ull); _Pragma(\"unroll\") for (int v = 0; v < V; ++v) {x}[v] = s; }}")
            return x
        m = self.map_of[k]
        if full and L.vec != 0:
            off = f"(ob{m} + rp{m})"
            if L.vec == 1:
                out.append(f"GFB_LOADV(B{k} + {off}, {x});")
            elif L.vec == 3:
                for v in range(V):
                    out.append(f"{x}[{v}] = GFB_LD(B{k} + (int32_t){off} + {L.dv[v]});")
            else:
                out.append(f"{{ const T s = GFB_LD(B{k} + {off}); _Pragma(\"unroll\") for (int v = 0; v < V; ++v) {x}[v] = s; }}")
            return x
        for v in range(V):
            e = f"GFB_LD(B{k} + ({self._elem(k, v)}))"
            out.append(f"{x}[{v}] = {e};" if full else f"{x}[{v}] = {v} < nvalid ? {e} : T(0);")
        return x

    def store(self, k, full, src, out):
        L, V = self.leaves[k], self.V
        m = self.map_of[k]
        if full and L.vec == 1:
            out.append(f"storeV<T, V>(B{k} + (ob{m} + rp{m}), {src});")
            return
        if full and L.vec == 3:
            for v in range(V):
                out.append(f"B{k}[(int32_t)(ob{m} + rp{m}) + {L.dv[v]}] = {src}[{v}];")
            return
        for v in range(V):
            st = f"B{k}[{self._elem(k, v)}] = {src}[{v}];"
            out.append(st if full else f"if ({v} < nvalid) {st}")

    # ---- the program (vm_run) --------------------------------------------
    def program(self, full):
        a, out = self.a, []
        for m in range(len(self.maps)):
            out.append(f"const uint32_t rp{m} = {self._rpart(m, 'r')};")
        pre = [self.load(k, full, out) for k in range(a.npre)]
        cache, stack, acc = {}, [], None

        def ld(k):
            if k not in cache:
                cache[k] = self.load(k, full, out)
            return cache[k]

        def new(expr):
            x = self._tmp()
            out.append(f"T {x}[V]; _Pragma(\"unroll\") for (int v = 0; v < V; ++v) {x}[v] = {expr};")
            return x

        for w in a.prog[:a.ninstr]:
            f, k, k2 = w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF
            if F_LOADP <= f < F_LOADP + 4:
                acc = pre[f - F_LOADP]
            elif f == F_LOADM:
                acc = ld(k)
            elif f == F_PUSH:
                stack.append(acc)
            elif f == F_STORE:
                self.store(k, full, acc, out)
                cache.clear()
            elif F_UN <= f < F_UN + 6:
                x = self._tmp()
                out.append(f"T {x}[V]; copyV<T, V>({x}, {acc}); apply_unary_c<{f - F_UN + 5}u, T, V>({x});")
                acc = x
            elif f == F_DOT:
                xa, xb = ld(k), ld(k2)
                acc = new(f"bin1<T>(0u, {acc}[v], bin1<T>(2u, {xa}[v], {xb}[v]))")
            elif f >= F_BIN:
                rel = f - F_BIN
                sw, rest = rel % 2, rel // 2
                src, op = rest // 5, rest % 5
                b = pre[src] if src < 4 else ld(k) if src == 4 else stack.pop() if src == 5 else acc
                acc = new(f"bin1<T>({op}u, {b}[v], {acc}[v])" if sw else f"bin1<T>({op}u, {acc}[v], {b}[v])")
            else:
                raise ValueError(f"bad VM word {w:#x}")
        if a.red_kind and acc is not None:  # (an empty program only occurs over an empty extent)
            out.append(f"copyV<T, V>(acc, {acc});")
        return out

    # ---- kernel ------------------------------------------------------------
    def emit(self):
        """The full translation unit of this launch alone."""
        return _kernel_source([self])

    def member(self, idx):
        """This launch as `namespace m<idx> { run(pa, dyn) }`."""
        a, V = self.a, self.V
        row = a.mode in (1, 3)
        n_o, n_r = a.n_o, a.n_r
        L = [f"namespace m{idx} {{", f"typedef {self.t} T;", f"constexpr int V = {V};",
             "__device__ __forceinline__ void run(const gfb_ew_args& pa, unsigned char* dyn) {"]
        L.append("const int nthr = blockDim.x, tid = threadIdx.x;")
        L.append("T* scratch = reinterpret_cast<T*>(dyn); (void)scratch;")
        for k, lf in enumerate(self.leaves):
            if lf.mode == 1:
                continue
            c = "" if k in self.stored else "const "
            L.append(f"{c}T* const B{k} = reinterpret_cast<{c}T*>(static_cast<{c}char*>(const_cast<void*>(pa.tab[{lf.ref >> 56}])) + "
                     f"{lf.ref & ((1 << 56) - 1)}ull);")
        kind = a.red_kind
        red = a.red_out
        if kind:
            L.append(f"T* const red = reinterpret_cast<T*>(reinterpret_cast<char*>(const_cast<void*>(pa.tab[{red.ref >> 56}])) + "
                     f"{red.ref & ((1 << 56) - 1)}ull);")
        red_digits = self._digits(red)[1] if kind else ()
        full_only = (n_r % V == 0) if row else (n_o % V == 0)
        body_full = self.program(True)
        body_part = None if full_only else self.program(False)

        def run(lines):
            if body_part is None:
                lines += ["{", *body_full, "}"]
            else:
                lines += ["if (nvalid == V) {", *body_full, "} else {", *body_part, "}"]

        ob = [f"const uint32_t ob{m} = {self._expr(self.maps[m][1], 'o', '0u', src=0)};" for m in range(len(self.maps))]
        if a.mode == 3:
            # chunk-wise (csrc/ew_vm.cu gfb_ew_staged_kernel, split == 1): a warp
            # per (o, chunk) item of CH elements; partial -> red[o * nch + chunk]
            # V here is one 16-byte piece (HV); the lane's pieces of a chunk are
            # (u, h) = 0..3 at chunk + (2u + h) * 32 * HV + lane * HV, folded in
            # (u, h, j) order exactly like the VM's sidx(u, h, lane, j)
            ch = 32 * 2 * (16 // self.esize) * 2  # StagedCfg<T, 2>::CH
            L += [
                "const int lane = tid & 31, warp = tid >> 5;",
                f"constexpr uint32_t CH = {ch}u, nr = {n_r}u, no = {n_o}u, nch = (nr + CH - 1) / CH;",
                "const uint32_t items = no * nch, wpb = nthr >> 5;",
                "for (uint32_t g = blockIdx.x * wpb + warp; g < items; g += gridDim.x * wpb) {",
                "const uint32_t o = g / nch, c = g % nch, rend = min(nr, (c + 1u) * CH);",
                f"T part = fold_init<T>({kind});",
                *ob,
                "_Pragma(\"unroll\") for (uint32_t piece = 0; piece < 4u; ++piece) {",
                "const uint32_t r = c * CH + piece * 32u * V + lane * V;",
                "if (r >= rend) continue;",
                "const int nvalid = (int)min((uint32_t)V, nr - r);",
            ]
            if kind:
                L.append("T acc[V];")
            run(L)
            if kind:
                L.append(f"_Pragma(\"unroll\") for (int v = 0; v < V; ++v) if (v < nvalid) part = fold<T>({kind}, part, acc[v]);")
            L.append("}")  # r loop
            if kind:
                L += [
                    f"_Pragma(\"unroll\") for (int off = 16; off > 0; off >>= 1) part = fold<T>({kind}, part, __shfl_xor_sync(0xffffffffu, part, off));",
                    "if (lane == 0) red[(size_t)o * nch + c] = part;",
                ]
            L.append("}")  # item loop
            smem = 0
        elif row:
            L += [
                "const int lane = tid & 31, warp = tid >> 5;",
                f"constexpr int wpr = {a.wpr};",
                "const int rpb = (nthr >> 5) / wpr;",
                "const int sub = warp % wpr, slot = warp / wpr;",
                f"constexpr uint32_t rstep = 32u * V * wpr, nr = {n_r}u, no = {n_o}u;",
                "for (uint32_t o0 = blockIdx.x * rpb; o0 < no; o0 += gridDim.x * rpb) {",
                "const uint32_t o = o0 + slot;",
                "const bool active = o < no;",
                f"T part = fold_init<T>({kind});",
                "if (active) {",
                *ob,
                "for (uint32_t rl = (sub * 32u + lane) * V; rl < nr; rl += rstep) {",
            ]
            if a.ty_ext:
                L += [
                    f"const uint32_t w = rl / V, xblocks = {a.ty_div}u / V;",
                    f"const uint32_t y = w % {a.ty_ext}u, t = w / {a.ty_ext}u;",
                    f"const uint32_t r = ((t / xblocks) * {a.ty_ext}u + y) * {a.ty_div}u + (t % xblocks) * V;",
                ]
            else:
                L.append("const uint32_t r = rl;")
            L.append("const int nvalid = (int)min((uint32_t)V, nr - r);")
            if kind:
                L.append("T acc[V];")
            run(L)
            if kind:
                L.append(f"_Pragma(\"unroll\") for (int v = 0; v < V; ++v) if (v < nvalid) part = fold<T>({kind}, part, acc[v]);")
            L += ["}", "}"]  # r loop, active
            if kind:
                roff = self._expr(red_digits, "o", "0u")
                L += [
                    f"_Pragma(\"unroll\") for (int off = 16; off > 0; off >>= 1) part = fold<T>({kind}, part, __shfl_xor_sync(0xffffffffu, part, off));",
                ]
                if a.wpr > 1:
                    L += [
                        "if (lane == 0) scratch[warp] = part;",
                        "__syncthreads();",
                        "if (active && sub == 0 && lane == 0) {",
                        f"for (int s = 1; s < wpr; ++s) part = fold<T>({kind}, part, scratch[warp + s]);",
                        f"red[{roff}] = part;",
                        "}",
                        "__syncthreads();",
                    ]
                else:
                    L.append(f"if (active && lane == 0) red[{roff}] = part;")
            L.append("}")  # o loop
            smem = (self.block // 32) * self.esize if (kind and a.wpr > 1) else 0
        else:
            L += [
                f"constexpr uint32_t split = {a.split}u, nr = {n_r}u, no = {n_o}u;",
                "const uint32_t per_row = nthr / split;",
                "const uint32_t lane_o = tid % per_row, rs = tid / per_row;",
                "const uint32_t o_stride = gridDim.x * per_row * V;",
                "for (uint32_t o0 = (blockIdx.x * per_row) * V; o0 < no; o0 += o_stride) {",
                "const uint32_t olin = o0 + lane_o * V;",
                "const bool active = olin < no;",
                "uint32_t o = olin;",
            ]
            if a.ty_ext:
                L += [
                    "if (active) {",
                    f"const uint32_t w = olin / V, xblocks = {a.ty_div}u / V;",
                    f"const uint32_t y = w % {a.ty_ext}u, t = w / {a.ty_ext}u, xb = t % xblocks, rest = t / xblocks;",
                    f"o = (rest * {a.ty_ext}u + y) * {a.ty_div}u + xb * V;",
                    "}",
                ]
            L += [
                "const int nvalid = active ? (int)min((uint32_t)V, no - o) : 0;",
                "T part[V];",
                f"_Pragma(\"unroll\") for (int v = 0; v < V; ++v) part[v] = fold_init<T>({kind});",
                "if (active) {",
                *ob,
                "for (uint32_t r = rs; r < nr; r += split) {",
            ]
            if kind:
                L.append("T acc[V];")
            run(L)
            if kind:
                L.append(f"_Pragma(\"unroll\") for (int v = 0; v < V; ++v) part[v] = fold<T>({kind}, part[v], acc[v]);")
            L += ["}", "}"]
            if kind:
                L.append("if (split > 1) {")
                L += [
                    "__syncthreads();",
                    "_Pragma(\"unroll\") for (int v = 0; v < V; ++v) scratch[v * nthr + tid] = part[v];",
                    "__syncthreads();",
                    "if (rs == 0) {",
                    "for (uint32_t s = 1; s < split; ++s)",
                    f"_Pragma(\"unroll\") for (int v = 0; v < V; ++v) part[v] = fold<T>({kind}, part[v], scratch[v * nthr + s * per_row + lane_o]);",
                    "}",
                    "}",
                    "if (active && rs == 0) {",
                ]
                each = (f"_Pragma(\"unroll\") for (int v = 0; v < V; ++v) if (v < nvalid) "
                        f"red[{self._expr(red_digits, 'o + v', '0u')}] = part[v];")
                if red.vec == 1:
                    L += [f"if (nvalid == V) {{ storeV<T, V>(red + ({self._expr(red_digits, 'o', '0u', src=0)}), part); }} else {{",
                          each, "}"]
                else:
                    L.append(each)
                L.append("}")
            L.append("}")  # o loop
            smem = V * self.block * self.esize if (kind and a.split > 1) else 0
        L.append("}")  # run
        L.append("}")  # namespace
        self.smem = smem
        return "\n".join(L) + "\n"

    @property
    def esize(self):
        return 8 if self.t == "double" else 4


def _headers_digest() -> str:
    global _header_digest
    if _header_digest is None:
        h = hashlib.sha256()
        for p in HEADERS:
            with open(p, "rb") as fh:
                h.update(fh.read())
        _header_digest = h.hexdigest()
    return _header_digest


def _cache_dir() -> str:
    d = os.environ.get("GFB_JIT_CACHE") or os.path.join(os.path.expanduser("~"), ".cache", "gfb200_jit")
    os.makedirs(d, exist_ok=True)
    return d


def compile_cubin(src: str) -> bytes:
    """NVRTC -> sm_100a cubin (disk-cached)."""
    key = hashlib.sha256((src + "\0" + " ".join(OPTIONS) + "\0" + _headers_digest()).encode()).hexdigest()
    path = os.path.join(_cache_dir(), key + ".cubin")
    if os.path.exists(path):
        with open(path, "rb") as fh:
            return fh.read()
    L = _lib_nvrtc()
    prog = C.c_void_p()
    rc = L.nvrtcCreateProgram(C.byref(prog), src.encode(), b"gfb_jit_ew.cu", 0, None, None)
    if rc:
        raise RuntimeError(f"nvrtcCreateProgram failed ({rc})")
    try:
        opts = OPTIONS + [f"-I{CSRC}", f"-I{INCLUDE}", f"-I{CUDA_INCLUDE}"]
        arr = (C.c_char_p * len(opts))(*[o.encode() for o in opts])
        rc = L.nvrtcCompileProgram(prog, len(opts), arr)
        if rc:
            n = C.c_size_t()
            L.nvrtcGetProgramLogSize(prog, C.byref(n))
            log = C.create_string_buffer(n.value)
            L.nvrtcGetProgramLog(prog, log)
            raise RuntimeError(f"NVRTC compile failed ({rc}):\n{log.value.decode(errors='replace')[-4000:]}")
        n = C.c_size_t()
        L.nvrtcGetCUBINSize(prog, C.byref(n))
        buf = C.create_string_buffer(n.value)
        L.nvrtcGetCUBIN(prog, buf)
        cubin = buf.raw
    finally:
        L.nvrtcDestroyProgram(C.byref(prog))
    tmp = f"{path}.{os.getpid()}.{threading.get_ident()}.tmp"
    with open(tmp, "wb") as fh:
        fh.write(cubin)
    os.replace(tmp, path)
    return cubin


def eligible(L) -> bool:
    return L.kind == abi.K_ROWJIT or (L.kind in KINDS and (L.algo_bytes or 0) >= MIN_BYTES)


def _kernel(lib, cubin: bytes):
    d = hashlib.sha256(cubin).hexdigest()
    with _lock:
        k = _kernels.get(d)
        if k is None:
            h = C.c_void_p()
            buf = C.create_string_buffer(cubin, len(cubin))
            rc = lib.gfb_kernel_load(buf, ENTRY, C.byref(h))
            if rc:
                raise RuntimeError(f"gfb_kernel_load failed: {lib.gfb_last_error().decode()}")
            k = _kernels[d] = h.value
    return k


MERGE = os.environ.get("GFB_JIT_MERGE", "1") == "1"


def _groups(launches, recs, todo):
    """Eligible launches in program order, consecutive single-block ones with
    the same block size merged into one group (they then run as one kernel
    with block barriers between them)."""
    groups, run = [], []
    prev = None
    for i in todo:
        r = recs[i]
        single = MERGE and tuple(r.grid) == (1, 1, 1) and launches[i].kind != abi.K_ROWJIT
        if single and run and prev == i - 1 and recs[run[0]].block[0] == r.block[0]:
            run.append(i)
        else:
            if run:
                groups.append(run)
            run = [i]
            if not single:
                groups.append(run)
                run = []
        prev = i
    if run:
        groups.append(run)
    return groups


def specialise(lib, handle, launches, blob: bytes, recs, workers: int | None = None):
    """Compile and install specialised kernels for the eligible launches of
    one executable.  Returns (indices of the launches replaced, indices of
    launches folded into a preceding merged kernel and skipped)."""
    todo = [i for i, L in enumerate(launches) if eligible(L)]
    if not todo:
        return [], []
    strict = os.environ.get("GFB_JIT_STRICT", "0") == "1"
    try:
        _lib_nvrtc()
    except RuntimeError as exc:
        if strict or any(launches[i].kind == abi.K_ROWJIT for i in todo):
            raise
        _warn_once(f"runtime specialisation off ({exc}); the generic VM kernel runs every elementwise launch")
        return [], []

    def args_of(i):
        r = recs[i]
        return abi.EwArgs.from_buffer_copy(blob[r.arg_offset:r.arg_offset + r.arg_size])

    def build(group):
        if launches[group[0]].kind == abi.K_ROWJIT:  # row-fused launch: generated or nothing (rowfuse.py)
            from .rowfuse import generate_source

            return group, compile_cubin(generate_source(launches[group[0]].row_spec)), 0
        if len(group) == 1:
            g = generate(launches[group[0]].kind, args_of(group[0]), recs[group[0]].block[0])
        else:
            g = generate_merged([(launches[i].kind, args_of(i)) for i in group], recs[group[0]].block[0])
        if g is None:
            return None
        try:
            return group, compile_cubin(g[0]), g[1]
        except RuntimeError as exc:  # a generator bug: keep the generic kernel, loudly
            if strict:
                raise
            _warn_once(f"{launches[group[0]].label}: specialised kernel failed to compile, generic kernel kept: {exc}")
            return None

    groups = _groups(launches, recs, todo)
    # a merged group that fails to generate falls back to its members one by one
    workers = workers or min(len(groups), max(1, (os.cpu_count() or 4)))
    with ThreadPoolExecutor(workers) as ex:
        built = list(ex.map(build, groups))
    retry = [[i] for grp, b in zip(groups, built) if b is None and len(grp) > 1 for i in grp]
    if retry:
        with ThreadPoolExecutor(workers) as ex:
            built += list(ex.map(build, retry))
    replaced, skipped = [], []
    for b in built:
        if b is None:
            continue
        group, cubin, smem = b
        rc = lib.gfb_exe_set_kernel(handle, group[0], C.c_void_p(_kernel(lib, cubin)), smem)
        if rc:
            raise RuntimeError(f"gfb_exe_set_kernel({group[0]}) failed: {lib.gfb_last_error().decode()}")
        replaced.append(group[0])
        for i in group[1:]:
            rc = lib.gfb_exe_set_kernel(handle, i, None, 0)  # runs inside the merged kernel
            if rc:
                raise RuntimeError(f"gfb_exe_set_kernel({i}, skip) failed: {lib.gfb_last_error().decode()}")
            skipped.append(i)
    return sorted(replaced), sorted(skipped)
