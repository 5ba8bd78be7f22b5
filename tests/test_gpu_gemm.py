"""tcgen05 3xTF32 Dot vs the oracle (normwise 1e-5)."""

import numpy as np
import pytest

import golden_io as G
from oracle import interp

pytestmark = pytest.mark.gpu
gf = pytest.importorskip("paper_1801_08058_b200")
K = gf.OpKind
F32 = gf.ElementType.F32


def _dot_graph(m, k, n, ta=False, tb=False):
    fn = gf.Function("dot")
    a = fn.add_parameter(F32, (k, m) if ta else (m, k))
    b = fn.add_parameter(F32, (n, k) if tb else (k, n))
    x = fn.add_node(K.RESHAPE, [a], {"input_order": (1, 0), "output_shape": (m, k)}) if ta else a
    y = fn.add_node(K.RESHAPE, [b], {"input_order": (1, 0), "output_shape": (k, n)}) if tb else b
    fn.set_results([fn.add_node(K.DOT, [x, y])])
    return fn


@pytest.mark.parametrize("m,k,n,ta,tb", [
    (128, 128, 128, False, False),
    (256, 512, 384, False, False),
    (130, 90, 70, False, False),
    (300, 777, 129, True, False),
    (257, 64, 511, False, True),
    (200, 301, 190, True, True),
    (1, 40, 3, False, False),
    (300, 600, 520, False, False),   # 2-SM pair kernel, ragged tiles
    (513, 4096, 256, False, True),   # pair kernel, long K (promotion chunks)
    (256, 20000, 256, True, False),  # pair kernel under split-K
])
def test_tc_dot_matches_oracle(monkeypatch, m, k, n, ta, tb):
    monkeypatch.setenv("GFB_DOT", "tc")
    monkeypatch.setenv("GFB_F16", "0")
    fn = _dot_graph(m, k, n, ta, tb)
    rng = np.random.default_rng(m * 7 + k + n)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    exe = gf.compile_function(fn)
    assert any("dot_tc" in L.label for L in exe.lowered.launches)
    out = gf.call(exe, [gf.tensor_from_flat(F32, a.shape, a) for a in ins])[0].to_numpy()
    want = interp.run_function(fn, ins)[0]
    err = G.normwise(out, want)
    assert err <= 1e-5, err


@pytest.mark.parametrize("m,k,n,ta,tb,et", [
    (1, 5, 5000, False, False, "F32"),
    (4, 6, 3001, False, False, "F32"),
    (8, 9, 700, True, False, "F32"),
    (3, 17, 1025, False, True, "F64"),
    (128, 512, 10, False, False, "F32"),   # thread-per-output kernel, A rows and B staged in shared memory
    (40, 33, 70, True, True, "F64"),
    (512, 128, 10, True, False, "F32"),    # the classifier's weight gradient (transposed A)
    (33, 300, 7, False, True, "F64"),
    (50, 4000, 8, False, False, "F32"),    # too big to stage: the register-pipelined form
])
def test_small_m_dot_bit_exact(m, k, n, ta, tb, et):
    """Few-row Dots with k > TINY_DOT_K take the thread-per-column SIMT
    kernel and keep the reference k order: bit-exact."""
    et = getattr(gf.ElementType, et)
    fn = gf.Function("dot")
    a = fn.add_parameter(et, (k, m) if ta else (m, k))
    b = fn.add_parameter(et, (n, k) if tb else (k, n))
    x = fn.add_node(K.RESHAPE, [a], {"input_order": (1, 0), "output_shape": (m, k)}) if ta else a
    y = fn.add_node(K.RESHAPE, [b], {"input_order": (1, 0), "output_shape": (k, n)}) if tb else b
    fn.set_results([fn.add_node(K.DOT, [x, y])])
    rng = np.random.default_rng(m + k + n)
    dt = et.numpy_dtype
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(dt) for p in fn.parameters]
    exe = gf.compile_function(fn)
    assert any(L.kind in (15, 16, 26, 27) for L in exe.lowered.launches)
    out = gf.call(exe, [gf.tensor_from_flat(et, v.shape, v) for v in ins])[0].to_numpy()
    assert G.same_bits(out, interp.run_function(fn, ins)[0])


def test_tc_dot_large_config_E_layer(monkeypatch):
    monkeypatch.setenv("GFB_F16", "0")
    fn = _dot_graph(2048, 4096, 4096)
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, size=(2048, 4096)).astype(np.float32)
    b = rng.uniform(-1 / 64, 1 / 64, size=(4096, 4096)).astype(np.float32)
    exe = gf.compile_function(fn)
    assert any("dot_tc" in L.label for L in exe.lowered.launches)
    out = gf.call(exe, [gf.tensor_from_flat(F32, a.shape, a), gf.tensor_from_flat(F32, b.shape, b)])[0].to_numpy()
    ref = (a.astype(np.float64) @ b.astype(np.float64))
    assert G.normwise(out, ref) <= 1e-5


@pytest.mark.parametrize("op,shape,stride,pad,layout", [
    ("fwd", (4, 3, 16, 32, 32, 3, 3), (1, 1), (1, 1, 1, 1), "identity"),
    ("fwd", (2, 16, 32, 33, 31, 3, 3), (2, 1), (0, 1, 1, 0), "identity"),
    ("fwd", (4, 16, 32, 32, 32, 3, 3), (1, 1), (1, 1, 1, 1), "nhwc"),
    ("dgrad", (4, 16, 32, 32, 32, 3, 3), (1, 1), (1, 0, 0, 1), "identity"),
    ("wgrad", (8, 16, 32, 32, 32, 3, 3), (1, 1), (1, 1, 1, 1), "identity"),
    ("wgrad", (8, 3, 16, 32, 32, 3, 3), (1, 1), (1, 1, 1, 1), "identity"),
    ("fwd", (4, 3, 64, 40, 40, 7, 7), (1, 1), (3, 3, 3, 3), "identity"),   # the config-D stem shape (stem kernel)
    ("wgrad", (4, 3, 64, 40, 40, 7, 7), (1, 1), (3, 3, 3, 3), "identity"),
    ("fwd", (2, 16, 32, 33, 31, 3, 3), (2, 1), (0, 1, 1, 0), "nhwc"),
    ("dgrad", (4, 16, 40, 20, 20, 3, 3), (1, 1), (1, 1, 1, 1), "identity"),
])
def test_conv_tensor_cores_match_oracle(monkeypatch, op, shape, stride, pad, layout):
    import test_lowering as TL

    monkeypatch.setenv("GFB_CONV", "tc")
    N, C, Ko, H, W, R, S = shape
    fn = TL._conv_graph(op, N, C, Ko, H, W, R, S, stride, pad)
    exe = gf.compile_function(fn, conv_layout=layout) if op == "fwd" else gf.compile_function(fn)
    assert any("_tc" in L.label or "_stem" in L.label for L in exe.lowered.launches)
    rng = np.random.default_rng(7)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(F32, v.shape, v, exe.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = gf.call(exe, tens)[0].to_numpy()
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("op,shape,stride,pad", [
    ("fwd", (4, 32, 64, 32, 32, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (2, 64, 96, 33, 31, 3, 3), (2, 2), (1, 1, 1, 1)),
    ("fwd", (3, 128, 256, 14, 14, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (2, 64, 128, 28, 28, 1, 1), (2, 2), (0, 0, 0, 0)),
    ("dgrad", (4, 40, 64, 16, 15, 3, 3), (1, 1), (1, 0, 0, 1)),
    ("dgrad", (2, 64, 128, 28, 28, 3, 3), (1, 1), (1, 1, 1, 1)),
    # channel counts that are multiples of 4 but not 32: K-blocks span taps
    ("fwd", (8, 16, 32, 32, 32, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (3, 4, 64, 30, 29, 7, 7), (1, 1), (3, 3, 3, 3)),
    ("fwd", (2, 12, 40, 17, 19, 3, 3), (2, 1), (0, 1, 1, 0)),
    ("dgrad", (4, 20, 16, 16, 15, 3, 3), (1, 1), (1, 0, 0, 1)),
    ("fwd", (4, 3, 64, 40, 36, 7, 7), (1, 1), (3, 3, 3, 3)),  # the stem: zero-padded to 4 channels
])
def test_conv_fused_gather_matches_oracle(monkeypatch, op, shape, stride, pad):
    """gfb_conv_tcg_kernel (in-kernel NHWC gather + TF32 split) vs the oracle."""
    import test_lowering as TL
    from paper_1801_08058_b200 import abi

    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_CONV_F16", "0")
    monkeypatch.setenv("GFB_PAD_CHANNELS_FWD", "1")
    monkeypatch.setenv("GFB_CONV_STEM", "0")
    N, C, Ko, H, W, R, S = shape
    fn = TL._conv_graph(op, N, C, Ko, H, W, R, S, stride, pad)
    nhwc = gf.Layout((0, 2, 3, 1))
    exe = gf.compile_function(fn, conv_layout="nhwc", parameter_layouts=[nhwc, None, nhwc][: len(fn.parameters)])
    assert any(L.kind in (abi.K_CONV_TCG64, abi.K_CONV_TCG128) for L in exe.lowered.launches)
    rng = np.random.default_rng(11)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(F32, v.shape, v, exe.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = gf.call(exe, tens)[0].to_numpy()
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("op,shape,stride,pad", [
    ("fwd", (4, 64, 64, 56, 56, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (3, 64, 96, 33, 31, 3, 3), (2, 2), (1, 1, 1, 1)),
    ("fwd", (5, 128, 256, 7, 7, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (2, 64, 128, 28, 28, 1, 1), (2, 2), (0, 0, 0, 0)),
    ("fwd", (2, 32, 128, 20, 3, 3, 3), (1, 2), (1, 1, 1, 1)),
    ("dgrad", (4, 40, 64, 16, 15, 3, 3), (1, 1), (1, 0, 0, 1)),
    ("dgrad", (2, 64, 128, 28, 28, 3, 3), (1, 1), (1, 1, 1, 1)),
])
def test_conv_tma_box_matches_oracle(monkeypatch, op, shape, stride, pad):
    """gfb_conv_tcx_kernel (TMA pixel-box gather, in-smem TF32 split) vs the oracle."""
    import test_lowering as TL  # noqa: F401  (shared helpers)
    from paper_1801_08058_b200 import abi

    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_CONV_F16", "0")
    Ko = gf.OpKind
    N, C, K, H, W, R, S = shape
    fn = gf.Function("conv")
    if op == "fwd":
        x = fn.add_parameter(F32, (N, C, H, W))
        f = fn.add_parameter(F32, (K, C, R, S))
        c = fn.add_node(Ko.CONV2D, [fn.add_node(Ko.RELU, [x]), f], {"strides": stride, "padding": pad})
    else:
        d = fn.add_parameter(F32, (N, K, H, W))
        f = fn.add_parameter(F32, (K, C, R, S))
        Hi, Wi = H - pad[0] - pad[1] + R - 1, W - pad[2] - pad[3] + S - 1
        c = fn.add_node(Ko.CONV_BACKPROP_DATA, [fn.add_node(Ko.RELU, [d]), f],
                        {"data_shape": (N, C, Hi, Wi), "padding": pad}, allow_internal=True)
    fn.set_results([fn.add_node(Ko.NEGATE, [c])])
    exe = gf.compile_function(fn, optimize=False, conv_layout="nhwc")
    assert any(L.kind in (abi.K_CONV_TCX64, abi.K_CONV_TCX128) for L in exe.lowered.launches)
    rng = np.random.default_rng(17)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    out = gf.call(exe, [gf.tensor_from_flat(F32, v.shape, v) for v in ins])[0].to_numpy()
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("m,k,n,et", [(2, 2, 2, "F64"), (1, 4, 4099, "F32"), (4, 1, 3001, "F32"), (2, 0, 3, "F64")])
def test_tiny_dot_fused_bit_exact_on_device(m, k, n, et):
    """Dots with k <= 4 run inside the VM kernel, bit-exact with the oracle."""
    et = getattr(gf.ElementType, et)
    fn = gf.Function("tiny")
    a = fn.add_parameter(et, (m, k))
    b = fn.add_parameter(et, (k, n))
    fn.set_results([fn.add_node(K.DOT, [a, b])])
    exe = gf.compile_function(fn, optimize=False)
    assert all(L.label.startswith("map:") for L in exe.lowered.launches)
    rng = np.random.default_rng(m + k + n)
    A = rng.uniform(-1, 1, size=(m, k)).astype(et.numpy_dtype)
    B = rng.uniform(-1, 1, size=(k, n)).astype(et.numpy_dtype)
    out = gf.call(exe, [gf.tensor_from_flat(et, A.shape, A), gf.tensor_from_flat(et, B.shape, B)])[0].to_numpy()
    assert G.same_bits(out, interp.run_function(fn, [A, B])[0])


@pytest.mark.parametrize("mn", [True, False])
@pytest.mark.parametrize("shape,pad", [((4, 64, 64, 28, 28, 3, 3), (1, 1, 1, 1)), ((2, 5, 16, 17, 15, 3, 3), (1, 0, 0, 1)),
                                       ((3, 12, 132, 9, 7, 3, 3), (1, 1, 0, 2)), ((2, 128, 256, 14, 14, 3, 3), (1, 1, 1, 1)),
                                       ((64, 64, 64, 16, 16, 1, 1), (0, 0, 0, 0)), ((8, 3, 64, 40, 36, 7, 7), (3, 3, 3, 3))])
def test_wgrad_channel_last_matches_oracle(monkeypatch, shape, pad, mn):
    """Weight gradient over channel-last data: the MN-major kernel (raw
    16-byte loads of x and dy, TF32 split in the kernel) and the generic
    element gather."""
    import test_lowering as TL
    from paper_1801_08058_b200 import abi

    monkeypatch.setenv("GFB_CONV_F16", "0")
    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_TCGW", "1" if mn else "0")
    N, C, Ko, H, W, R, S = shape
    fn = TL._conv_graph("wgrad", N, C, Ko, H, W, R, S, (1, 1), pad)
    nhwc = gf.Layout((0, 2, 3, 1))
    exe = gf.compile_function(fn, conv_layout="nhwc", parameter_layouts=[nhwc, None, nhwc])
    used = any(L.kind in (abi.K_CONV_TCGW64, abi.K_CONV_TCGW128) for L in exe.lowered.launches)
    assert used == (mn and Ko % 4 == 0 and (C % 4 == 0 or C < 32)), [L.label for L in exe.lowered.launches]
    rng = np.random.default_rng(23)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(F32, v.shape, v, exe.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = gf.call(exe, tens)[0].to_numpy()
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("shape,pad,layout", [
    ((4, 3, 64, 40, 36, 7, 7), (3, 3, 3, 3), "identity"),   # the ResNet stem, NCHW input
    ((2, 3, 16, 32, 32, 3, 3), (1, 1, 1, 1), "identity"),   # config C's first layer (16 < 64 columns)
    ((3, 4, 64, 17, 23, 5, 5), (2, 1, 0, 3), "nhwc"),       # channel-last input, partial tiles
    ((2, 1, 40, 9, 11, 3, 3), (0, 0, 1, 1), "identity"),    # one channel, no padding rows
])
def test_conv_stem_kernel_matches_oracle(monkeypatch, shape, pad, layout):
    """gfb_conv_stem_kernel (8x16 pixel tiles from a shared-memory input
    patch, resident filter planes) vs the oracle."""
    import test_lowering as TL
    from paper_1801_08058_b200 import abi

    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_CONV_F16", "0")
    N, C, Ko, H, W, R, S = shape
    fn = TL._conv_graph("fwd", N, C, Ko, H, W, R, S, (1, 1), pad)
    lay = [gf.Layout((0, 2, 3, 1)), None] if layout == "nhwc" else None
    exe = gf.compile_function(fn, conv_layout=layout, parameter_layouts=lay)
    assert any(L.kind == abi.K_CONV_STEM64 for L in exe.lowered.launches), [L.label for L in exe.lowered.launches]
    rng = np.random.default_rng(31)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(F32, v.shape, v, exe.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = gf.call(exe, tens)[0].to_numpy()
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("shape,pad,layout", [
    ((4, 3, 64, 40, 36, 7, 7), (3, 3, 3, 3), "identity"),   # the ResNet stem, NCHW input
    ((2, 3, 16, 32, 32, 3, 3), (1, 1, 1, 1), "identity"),   # config C's first layer (16 < 64 columns)
    ((3, 4, 64, 17, 23, 5, 5), (2, 1, 0, 3), "nhwc"),       # channel-last input, partial tiles
    ((2, 1, 40, 9, 11, 3, 3), (0, 0, 1, 1), "identity"),    # one channel, no padding rows
    ((2, 3, 48, 20, 19, 8, 8), (4, 3, 3, 4), "nhwc"),       # K = 192: three full K-blocks
    ((37, 3, 64, 24, 24, 7, 7), (3, 3, 3, 3), "nhwc"),      # more tiles than CTAs: the persistent walk
])
def test_conv_stemh_kernel_matches_oracle(monkeypatch, shape, pad, layout):
    """gfb_conv_stemh_kernel (the stem's tiles in 2xFP16: per-tile activation
    scales, the filter split in the prologue) vs the oracle, with inputs
    whose magnitude varies by 10^6 between images and tiles (GFB_STEMH_ALL:
    also the shapes that default to the TF32 stem kernel)."""
    import test_lowering as TL
    from paper_1801_08058_b200 import abi

    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_STEMH_ALL", "1")
    N, C, Ko, H, W, R, S = shape
    fn = TL._conv_graph("fwd", N, C, Ko, H, W, R, S, (1, 1), pad)
    lay = [gf.Layout((0, 2, 3, 1)), None] if layout == "nhwc" else None
    exe = gf.compile_function(fn, conv_layout=layout, parameter_layouts=lay)
    assert any(L.kind in (abi.K_CONV_STEMH, abi.K_CONV_STEMH_C3R7) for L in exe.lowered.launches), \
        [L.label for L in exe.lowered.launches]
    rng = np.random.default_rng(37)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0][0] *= np.float32(1e-6)
    ins[0][:, :, : H // 3] *= np.float32(1e3)
    tens = [gf.tensor_from_flat(F32, v.shape, v, exe.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = gf.call(exe, tens)[0].to_numpy()
    interp.set_threads(interp.max_threads())
    ref = interp.run_function(fn, ins)[0]
    assert G.normwise(out, ref) <= 1e-5
    assert G.normwise(out[0], ref[0]) <= 1e-5  # the 1e-6 image on its own scale


@pytest.mark.parametrize("shape,pad,xlay", [
    ((2, 3, 64, 64, 64, 7, 7), (3, 3, 3, 3), "identity"),     # fewer tiles than CTAs
    ((4, 3, 64, 112, 112, 7, 7), (3, 3, 3, 3), "identity"),   # D's stem at half resolution, NCHW image
    ((3, 3, 64, 37, 45, 7, 7), (2, 4, 3, 1), "nhwc"),         # partial 2 x 32 tiles, asymmetric padding
])
def test_conv_stemwh_kernel_matches_oracle(monkeypatch, shape, pad, xlay):
    """gfb_conv_stemwh_kernel (the 3-channel 7x7 weight gradient in 2xFP16,
    per-tile scales promoted per tile, per-CTA partials) vs the oracle, with
    x and dy magnitudes varying by 10^6 between images and tiles."""
    import test_lowering as TL
    from paper_1801_08058_b200 import abi

    monkeypatch.setenv("GFB_CONV", "tc")
    N, C, Ko, H, W, R, S = shape
    fn = TL._conv_graph("wgrad", N, C, Ko, H, W, R, S, (1, 1), pad)
    nhwc = gf.Layout((0, 2, 3, 1))
    exe = gf.compile_function(fn, parameter_layouts=[nhwc if xlay == "nhwc" else None, None, nhwc])
    assert any(L.kind == abi.K_CONV_STEMWH_C3R7 for L in exe.lowered.launches), [L.label for L in exe.lowered.launches]
    rng = np.random.default_rng(41)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0][0] *= np.float32(1e-3)
    ins[2][-1] *= np.float32(1e3)
    ins[2][:, :, : H // 4] *= np.float32(1e-3)
    tens = [gf.tensor_from_flat(F32, v.shape, v, exe.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = gf.call(exe, tens)[0].to_numpy()
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("m,k,n", [(512, 4096, 256), (288, 1000, 352), (4096, 2048, 4096)])
@pytest.mark.parametrize("raw", ["mn", "kmajor", "split"])
def test_raw_hi_operands(monkeypatch, m, k, n, raw):
    """Arena-resident operands read in place as the tf32 hi operand (the MMA
    truncates), with one shared lo plane: K-major (Dot(h, W)) and MN-major
    via TMA SWIZZLE_128B_ATOM_32B (the weight gradient Dot(h^T, dz)),
    against the plane-split form and the oracle."""
    monkeypatch.setenv("GFB_F16", "0")
    if raw == "split":
        monkeypatch.setenv("GFB_RAW_HI", "0")
        monkeypatch.setenv("GFB_MN_MAJOR", "0")
    fn = gf.Function("raw")
    h = fn.add_parameter(F32, (k, m))
    dz = fn.add_parameter(F32, (k, n))
    rh, rd = fn.add_node(K.RELU, [h]), fn.add_node(K.NEGATE, [dz])  # arena-resident producers
    if raw == "kmajor":
        w = fn.add_parameter(F32, (m, n))
        out = fn.add_node(K.DOT, [rh, w])  # [k, m] x [m, n]: A K-major
    else:
        ht = fn.add_node(K.RESHAPE, [rh], {"input_order": (1, 0), "output_shape": (m, k)})
        out = fn.add_node(K.DOT, [ht, rd])  # [m, k] x [k, n]: both MN-major
    # rh's second reader keeps it materialised in the arena (as in config E,
    # where an activation feeds the next layer's Dot and this layer's weight
    # gradient); the transposing Reshape is then a free view
    fn.set_results([out, fn.add_node(K.SUM, [rh], {"reduction_axes": (0,)})])
    rng = np.random.default_rng(m + k + n)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    exe = gf.compile_function(fn)
    tc = [L for L in exe.lowered.launches if L.label.startswith("dot_tc")]
    assert tc
    if raw == "mn":
        assert tc[0].args.a_ld_mn == m and tc[0].args.b_ld_mn == n
        assert not any(L.label.startswith("split") for L in exe.lowered.launches)
    out = gf.call(exe, [gf.tensor_from_flat(F32, a.shape, a) for a in ins])[0].to_numpy()
    interp.set_threads(interp.max_threads())
    want = interp.run_function(fn, ins)[0]
    exact = np.maximum(ins[0].astype(np.float64), 0).T @ (-ins[1].astype(np.float64)) if raw != "kmajor" else \
        np.maximum(ins[0].astype(np.float64), 0) @ ins[2].astype(np.float64)
    assert G.normwise(out, exact) <= 1e-5 and G.normwise(out, want) <= 1e-5


@pytest.mark.parametrize("width,batch", [(512, 1024), (768, 2048)])
def test_fused_epilogues_bit_identical(monkeypatch, width, batch):
    """Bias + Relu after the forward Dot and the Relu-gradient mask after the
    data-gradient Dot, applied in the pair GEMM's epilogue: the same IEEE ops
    on the same accumulator values -> every result bit-identical to the plan
    that runs them as separate maps."""
    from paper_1801_08058_b200 import workloads as W

    monkeypatch.setenv("GFB_F16", "0")
    step = W.wide_mlp_step(gf, batch=batch, width=width, layers=3, loss_batch=65536)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=6, x_range=(-1, 1))
    tens = [gf.tensor_from_flat(F32, a.shape, a) for a in arrays]
    monkeypatch.setenv("GFB_TC_EPILOGUE", "1")
    exe = gf.compile_function(step.fn)
    from paper_1801_08058_b200 import abi

    kinds = {L.args.epi_kind for L in exe.lowered.launches if L.kind == abi.K_DOT_TC32P}
    assert kinds == {0, 1, 2}
    fused = [t.to_numpy() for t in gf.call(exe, tens)]
    monkeypatch.setenv("GFB_TC_EPILOGUE", "0")
    plain = [t.to_numpy() for t in gf.call(gf.compile_function(step.fn), tens)]
    for a, b in zip(fused, plain):
        assert G.same_bits(a, b)


# ---- 2xFP16 block-scaled pair GEMM (csrc/gemm_f16.cu) ----

@pytest.mark.parametrize("m,k,n,ta,tb", [
    (512, 1024, 512, False, False),   # A K-major, B MN-major (Dot(h, W))
    (512, 1024, 512, True, False),    # both MN-major (the weight gradient Dot(h^T, dz))
    (512, 1024, 512, False, True),    # both K-major (the data gradient Dot(dz, W^T))
    (512, 1024, 512, True, True),
    (320, 200, 256, False, False),    # ragged K (zero-filled TMA tail), ragged M tile
    (300, 600, 520, False, True),     # ragged tiles (K-major operands only: MN-major needs rows % 64)
    (256, 20000, 256, True, False),   # split-K on 128-K scale blocks
    (2048, 4096, 4096, False, False), # a config-E layer
])
def test_f16_dot_matches_exact(m, k, n, ta, tb):
    """fp16 hi / lo planes with 128 x 128 tile scales and three kind::f16
    MMAs per K-step: normwise within 1e-6 of the exact product (the Dot
    contract is 1e-5), including tiles whose magnitudes differ by 1e40."""
    fn = _dot_graph(m, k, n, ta, tb)
    rng = np.random.default_rng(m + 3 * k + n)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0].reshape(-1)[: 128 * 128] *= np.float32(1e-20)
    ins[1].reshape(-1)[-1000:] *= np.float32(1e20)
    exe = gf.compile_function(fn)
    from paper_1801_08058_b200 import abi

    assert [L.kind for L in exe.lowered.launches if L.flops] == [abi.K_DOT_F16P]
    out = gf.call(exe, [gf.tensor_from_flat(F32, a.shape, a) for a in ins])[0].to_numpy()
    A = ins[0].astype(np.float64).T if ta else ins[0].astype(np.float64)
    B = ins[1].astype(np.float64).T if tb else ins[1].astype(np.float64)
    ref = A @ B
    assert G.normwise(out, ref) <= 1e-6, G.normwise(out, ref)
    rows = 128 if not ta else m  # the scaled-down block's rows stand on their own
    assert G.normwise(out[:rows], ref[:rows]) <= 1e-6


@pytest.mark.parametrize("width,batch", [(512, 1024), (768, 2048)])
def test_f16_epilogue_planes_bit_identical(monkeypatch, width, batch):
    """The fp16 planes the fused epilogues write (block maximum, scale, hi /
    lo of the Relu output and of the masked gradient) equal the split pass
    over the unfused maps' results: every step result bit-identical."""
    from paper_1801_08058_b200 import abi, workloads as W

    step = W.wide_mlp_step(gf, batch=batch, width=width, layers=3, loss_batch=65536)
    arrays = W.step_inputs(step, W.parameter_shapes(step), seed=6, x_range=(-1, 1))
    tens = [gf.tensor_from_flat(F32, a.shape, a) for a in arrays]
    monkeypatch.setenv("GFB_TC_EPILOGUE", "1")
    exe = gf.compile_function(step.fn)
    f16 = [L for L in exe.lowered.launches if L.kind == abi.K_DOT_F16P]
    assert {L.args.epi_kind for L in f16} == {0, 1, 2} and any(L.args.epi_flags & 4 for L in f16)
    fused = [t.to_numpy() for t in gf.call(exe, tens)]
    monkeypatch.setenv("GFB_TC_EPILOGUE", "0")
    plain = [t.to_numpy() for t in gf.call(gf.compile_function(step.fn), tens)]
    for a, b in zip(fused, plain):
        assert G.same_bits(a, b)
    monkeypatch.setenv("GFB_F16", "0")
    tf32 = [t.to_numpy() for t in gf.call(gf.compile_function(step.fn), tens)]
    for a, b in zip(fused, tf32):
        assert G.normwise(a, b) <= 1e-5


@pytest.mark.parametrize("op,shape,stride,pad", [
    ("fwd", (4, 64, 64, 32, 32, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (3, 64, 96, 19, 17, 3, 3), (2, 2), (1, 1, 1, 1)),
    ("fwd", (2, 128, 256, 14, 14, 1, 1), (2, 2), (0, 0, 0, 0)),
    ("fwd", (2, 256, 128, 14, 14, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("dgrad", (4, 40, 64, 16, 15, 3, 3), (1, 1), (1, 0, 0, 1)),
    ("dgrad", (2, 64, 128, 14, 14, 3, 3), (1, 1), (1, 1, 1, 1)),
])
def test_conv_tcxh_matches_oracle(monkeypatch, op, shape, stride, pad):
    """2xFP16 TMA-box convolution (conv_f16.cu): channel-scaled fp16
    activation planes and filter planes divided by the same scales, channels
    1e20 apart: normwise within the 1e-5 Conv contract of the oracle (whose
    own sequential fp32 sums carry ~1e-6 of rounding at these depths)."""
    import test_lowering as TL
    from paper_1801_08058_b200 import abi

    monkeypatch.setenv("GFB_CONV", "tc")
    fn = TL._conv_fn(gf, op, shape, stride, pad)
    exe = gf.compile_function(fn, conv_layout="nhwc", optimize=False)
    assert any(L.kind in (abi.K_CONV_TCXH64, abi.K_CONV_TCXH128) for L in exe.lowered.launches)
    rng = np.random.default_rng(19)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0][:, 1] *= np.float32(1e-12)
    ins[0][:, 2] *= np.float32(1e8)
    out = gf.call(exe, [gf.tensor_from_flat(F32, v.shape, v) for v in ins])[0].to_numpy()
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("shape,pad", [
    ((8, 64, 64, 28, 28, 3, 3), (1, 1, 1, 1)),
    ((4, 128, 256, 14, 14, 1, 1), (0, 0, 0, 0)),
    ((4, 64, 128, 15, 13, 3, 3), (1, 0, 0, 1)),
    ((2, 512, 512, 7, 7, 3, 3), (1, 1, 1, 1)),
])
def test_conv_tcgwh_matches_oracle(monkeypatch, shape, pad):
    """2xFP16 weight gradient (conv_f16.cu gfb_conv_tcgwh_kernel) on the
    channel-scaled planes of x and dy vs the oracle: normwise within the 1e-5
    Conv contract (a contraction over up to 6272 pixels)."""
    from paper_1801_08058_b200 import abi

    monkeypatch.setenv("GFB_CONV", "tc")
    Ko = gf.OpKind
    N, C, K, H, W, R, S = shape
    fn = gf.Function("wgrad")
    x = fn.add_parameter(F32, (N, C, H, W))
    Ho, Wo = H + pad[0] + pad[1] - R + 1, W + pad[2] + pad[3] - S + 1
    d = fn.add_parameter(F32, (N, K, Ho, Wo))
    g = fn.add_node(Ko.CONV_BACKPROP_FILTER, [fn.add_node(Ko.RELU, [x]), fn.add_node(Ko.NEGATE, [d])],
                    {"filter_shape": (K, C, R, S), "padding": pad}, allow_internal=True)
    fn.set_results([g])
    exe = gf.compile_function(fn, conv_layout="nhwc", optimize=False)
    assert any(L.kind in (abi.K_CONV_TCGWH64, abi.K_CONV_TCGWH128) for L in exe.lowered.launches)
    rng = np.random.default_rng(29)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0][:, 3] *= np.float32(1e-9)
    out = gf.call(exe, [gf.tensor_from_flat(F32, v.shape, v) for v in ins])[0].to_numpy()
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


def test_f16_dot_special_values():
    """inf / NaN operands on the fp16 GEMM: the scales count finite values
    only, so exactly the outputs the reference makes non-finite are
    non-finite, and every other output stays within the Dot contract.  (An
    inf operand can give NaN where the reference has +-inf: the split's
    cross products multiply it by a zero lo part -- as in the 3xTF32
    kernel.)"""
    m, k, n = 512, 512, 512
    fn = _dot_graph(m, k, n)
    rng = np.random.default_rng(31)
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32) * np.float32(1e3)
    b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    a[5, 7] = np.inf
    a[300, 2] = np.nan
    b[9, 400] = -np.inf
    out = gf.call(gf.compile_function(fn), [gf.tensor_from_flat(F32, a.shape, a), gf.tensor_from_flat(F32, b.shape, b)])[0]
    out = out.to_numpy()
    with np.errstate(all="ignore"):
        ref = a.astype(np.float64) @ b.astype(np.float64)
    bad = ~np.isfinite(ref)
    assert np.array_equal(~np.isfinite(out), bad)
    good = ~bad
    assert G.normwise(out[good], ref[good]) <= 1e-6
