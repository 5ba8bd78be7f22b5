"""Fusion / index-map lowering checked on the host emulator against goldens.

The emulator executes the exact launch argument blocks the B200 receives
(magic-number digit maps, VM programs, strides) with sequential folds, so
every corpus graph must reproduce the reference interpreter's optimised
outputs.  F32 results must be bit-identical; F64 results may differ only
through libm-vs-numpy transcendentals (<= 1e-12, the reference corpus
tolerance, `_graphgen.tolerance_for`).
"""

import numpy as np
import pytest

import golden_io as G
from hostcompile import emulate, host_compile
from paper_1801_08058_b200 import abi


def _compare(outs, want_docs, label):
    for o, w in zip(outs, want_docs):
        w = G.logical(w)
        if w.dtype == np.float64:
            assert G.max_abs_diff(o, w) <= 1e-12, (label, o, w)
        else:
            assert G.same_bits(o, w), (label, o, w)


@pytest.mark.parametrize("seed", range(200))
def test_corpus_emulated(seed):
    case = G.load("corpus.json.gz")[seed]
    fn = G.fn_of(case["fn"])
    tensors = [G.tensor_of(d) for d in case["inputs"]]
    h = host_compile(fn)
    _compare(emulate(h, tensors), case["outputs_opt"], seed)
    h2 = host_compile(fn, optimize=False, private=(seed % 2 == 0))
    _compare(emulate(h2, tensors), case["outputs_noopt"], seed)


@pytest.mark.parametrize("seed", range(200))
def test_listing_matches_reference(seed):
    case = G.load("corpus.json.gz")[seed]
    fn = G.fn_of(case["fn"])
    assert host_compile(fn).listing() == case["listing_opt"]
    assert host_compile(fn, optimize=False).listing() == case["listing_noopt"]


@pytest.mark.parametrize("idx", range(12))
def test_layout_cases(idx):
    case = G.load("layouts.json.gz")[idx]
    fn = G.fn_of(case["fn"])
    h = host_compile(fn, optimize=case["conv_layout"] != "identity" or case["parameter_layouts"] is None,
                     conv_layout=case["conv_layout"], parameter_layouts=case["parameter_layouts"])
    if case["parameter_layouts"] is not None:
        h = host_compile(fn, optimize=False, parameter_layouts=case["parameter_layouts"])
    assert h.listing() == case["listing"]
    _compare(emulate(h, [G.tensor_of(d) for d in case["inputs"]]), case["outputs"], case["name"])


@pytest.mark.parametrize("name", ["mlp_A_small", "mlp_E_small", "cnn_C_small", "mlp_A_f64", "chain_B_small", "resnet_D_small"])
def test_workloads_emulated(name):
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == name)
    fn = G.fn_of(case["fn"])
    h = host_compile(fn)
    assert h.listing() == case["listing"]
    _compare(emulate(h, [G.tensor_of(d) for d in case["inputs"]]), case["outputs"], name)


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True)])
def test_tensor_core_lowering_emulated(monkeypatch, ta, tb):
    """Split planes + 3xTF32 product, emulated: normwise within 1e-5."""
    import paper_1801_08058_b200 as gf
    from oracle import interp

    monkeypatch.setenv("GFB_DOT", "tc")
    m, k, n = 37, 70, 45
    fn = gf.Function("dot")
    K, F32 = gf.OpKind, gf.ElementType.F32
    a = fn.add_parameter(F32, (k, m) if ta else (m, k))
    b = fn.add_parameter(F32, (n, k) if tb else (k, n))
    x = fn.add_node(K.RESHAPE, [a], {"input_order": (1, 0), "output_shape": (m, k)}) if ta else a
    y = fn.add_node(K.RESHAPE, [b], {"input_order": (1, 0), "output_shape": (k, n)}) if tb else b
    fn.set_results([fn.add_node(K.DOT, [x, y])])
    h = host_compile(fn)
    assert [L.label.split("#")[0] for L in h.lowered.launches] == ["split_a", "split_b", "dot_tc"]
    rng = np.random.default_rng(1)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    out = emulate(h, [gf.tensor_from_flat(F32, v.shape, v) for v in ins])[0]
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-6


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_f16_gemm_lowering_emulated(ta, tb):
    """fp16 planes with 128 x 128 tile scales + the 2xFP16 product (K-major
    and MN-major operands), emulated: normwise within 1e-6 of the oracle."""
    import paper_1801_08058_b200 as gf
    from oracle import interp

    m, k, n = 320, 200, 256
    fn = gf.Function("dot")
    K, F32 = gf.OpKind, gf.ElementType.F32
    a = fn.add_parameter(F32, (k, m) if ta else (m, k))
    b = fn.add_parameter(F32, (n, k) if tb else (k, n))
    x = fn.add_node(K.RESHAPE, [a], {"input_order": (1, 0), "output_shape": (m, k)}) if ta else a
    y = fn.add_node(K.RESHAPE, [b], {"input_order": (1, 0), "output_shape": (k, n)}) if tb else b
    fn.set_results([fn.add_node(K.DOT, [x, y])])
    h = host_compile(fn)
    labels = [L.label.split("#")[0] for L in h.lowered.launches]
    assert labels == ["split16", "split16", "dot_f16"], labels
    g = next(L.args for L in h.lowered.launches if L.kind == abi.K_DOT_F16P)
    assert (g.a_ld_mn > 0, g.b_ld_mn > 0) == (ta, not tb)
    rng = np.random.default_rng(1)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0][:128, :128] *= np.float32(1e-20)  # a tile far below the others: scales are per tile
    out = emulate(h, [gf.tensor_from_flat(F32, v.shape, v) for v in ins])[0]
    ref = interp.run_function(fn, ins)[0]
    assert G.normwise(out, ref) <= 1e-6
    assert G.normwise(out[:128], ref[:128]) <= 1e-6


def test_f16_epilogue_planes_emulated():
    """An MLP step whose hidden layers run on the fp16 GEMM: the bias + Relu
    and Relu-gradient epilogues write the next GEMMs' fp16 planes (no split
    pass for the activations); outputs within 1e-5 of the oracle."""
    import paper_1801_08058_b200 as gf
    from oracle import interp
    from paper_1801_08058_b200 import workloads as W

    st = W.mlp_step(gf, batch=256, in_dim=256, hidden=(256, 256), out_dim=256)
    h = host_compile(st.fn)
    labels = [L.label for L in h.lowered.launches]
    assert sum(lb.startswith("dot_f16") for lb in labels) == 8, labels  # 3 forward, 3 weight, 2 data gradients
    assert any("epibias_relu" in lb for lb in labels) and any("epirelu_grad" in lb for lb in labels)
    f16 = [L for L in h.lowered.launches if L.kind == abi.K_DOT_F16P]
    assert sum(1 for L in f16 if L.args.epi_flags & 4) >= 3
    # the backward reads the forward's mask bytes; the pre-activations and the
    # Relu outputs are then never stored (their readers take planes / masks)
    assert sum(1 for L in f16 if L.args.epi_flags & 8) == 2 and sum(1 for L in f16 if L.args.epi_flags & 16) == 2
    assert all(L.args.epi_flags & 32 and not L.args.epi_flags & 1 for L in f16 if L.args.epi_kind == 1)
    # the bias gradients reduce the Relu-gradient epilogues' 32-row column partials
    assert sum(1 for L in f16 if L.args.epi_flags & 64) == 2 and sum(":part" in lb for lb in labels) == 2
    rng = np.random.default_rng(3)
    ins = W.step_inputs(st, W.parameter_shapes(st), seed=3)
    out = emulate(h, [gf.tensor_from_flat(gf.ElementType.F32, v.shape, v) for v in ins])
    ref = interp.run_function(st.fn, ins)
    for o, r in zip(out, ref):
        assert G.normwise(o, r) <= 1e-5


@pytest.mark.parametrize("shape,axes", [((3, 5000), (1,)), ((2, 300, 40), (1, 2)), ((70000,), (0,))])
def test_chunkwise_reduction_emulated(shape, axes, monkeypatch):
    """Few long rows: staged chunk-wise partials + a second pass (the row
    fusion would otherwise take [3, 5000]: a small graph)."""
    monkeypatch.setenv("GFB_ROWFUSE", "0")
    import paper_1801_08058_b200 as gf
    from oracle import interp

    K, F32 = gf.OpKind, gf.ElementType.F32
    fn = gf.Function("red")
    x = fn.add_parameter(F32, shape)
    e = fn.add_node(K.EXP, [x])
    fn.set_results([fn.add_node(K.SUM, [e], {"reduction_axes": axes}), fn.add_node(K.NEGATE, [e])])
    h = host_compile(fn)
    labels = [L.label for L in h.lowered.launches]
    assert any(":pass2" in l for l in labels), labels
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, size=shape).astype(np.float32)
    outs = emulate(h, [gf.tensor_from_flat(F32, shape, v)])
    want = interp.run_function(fn, [v])
    assert G.normwise(outs[0], want[0]) <= 1e-5  # reduction order differs from the reference
    assert G.same_bits(outs[1], want[1])


def _conv_graph(op, N, C, K, H, W, R, S, stride=(1, 1), pad=(1, 1, 1, 1)):
    import paper_1801_08058_b200 as gf

    Ko, F32 = gf.OpKind, gf.ElementType.F32
    fn = gf.Function("conv")
    x = fn.add_parameter(F32, (N, C, H, W))
    f = fn.add_parameter(F32, (K, C, R, S))
    c = fn.add_node(Ko.CONV2D, [x, f], {"strides": stride, "padding": pad})
    if op == "fwd":
        fn.set_results([c])
        return fn
    d = fn.add_parameter(F32, fn.nodes[c].output.shape)
    if op == "dgrad":
        fn.set_results([fn.add_node(Ko.CONV_BACKPROP_DATA, [d, f], {"data_shape": (N, C, H, W), "padding": pad}, allow_internal=True)])
    else:
        fn.set_results([fn.add_node(Ko.CONV_BACKPROP_FILTER, [x, d], {"filter_shape": (K, C, R, S), "padding": pad}, allow_internal=True)])
    return fn


@pytest.mark.parametrize("op,shape,stride,pad,layout", [
    ("fwd", (2, 3, 8, 9, 10, 3, 3), (1, 1), (1, 1, 1, 1), "identity"),
    ("fwd", (2, 3, 9, 9, 10, 3, 2), (2, 1), (0, 1, 1, 0), "identity"),
    ("fwd", (2, 3, 8, 9, 10, 3, 3), (1, 1), (1, 1, 1, 1), "nhwc"),
    ("dgrad", (2, 5, 6, 7, 9, 3, 3), (1, 1), (1, 0, 0, 1), "identity"),
    ("wgrad", (2, 4, 6, 32, 32, 3, 3), (1, 1), (1, 1, 1, 1), "identity"),
    ("fwd", (2, 3, 16, 12, 12, 7, 7), (1, 1), (3, 3, 3, 3), "identity"),    # stem-like, generic gather
    ("wgrad", (2, 3, 16, 12, 12, 7, 7), (1, 1), (3, 3, 3, 3), "identity"),
    ("dgrad", (2, 6, 16, 9, 9, 3, 3), (1, 1), (1, 1, 1, 1), "identity"),
])
def test_conv_tensor_core_lowering_emulated(monkeypatch, op, shape, stride, pad, layout):
    """Implicit-GEMM convolutions (gather-split planes + 3xTF32 GEMM, split-K
    for the weight gradient), emulated, within 1e-5 normwise of the oracle."""
    import paper_1801_08058_b200 as gf
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    N, C, K, H, W, R, S = shape
    fn = _conv_graph(op, N, C, K, H, W, R, S, stride, pad)
    h = host_compile(fn, optimize=False, conv_layout=layout) if op == "fwd" else host_compile(fn, optimize=False)
    labels = [L.label for L in h.lowered.launches]
    assert any("_tc" in l or "_stem" in l for l in labels), labels
    if op == "fwd" and C < 16 and stride == (1, 1):  # few channels: the patch-staged stem kernels
        assert any(("_stemh#" if (C, R, S) == (3, 7, 7) else "_stem#") in l for l in labels), labels
    if op == "wgrad" and N * H * W >= 2048:  # long K: split-K with a deterministic second pass
        assert any(":splitk" in l for l in labels), labels
    rng = np.random.default_rng(5)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(gf.ElementType.F32, v.shape, v, h.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = emulate(h, tens)[0]
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("shape,pad,layout", [
    ((2, 3, 64, 12, 20, 7, 7), (3, 3, 3, 3), "identity"),  # the ResNet stem shape, partial tiles
    ((2, 3, 40, 9, 11, 8, 8), (4, 3, 3, 4), "nhwc"),       # K = 192 (three full K-blocks), 40 columns
    ((1, 1, 16, 10, 17, 3, 3), (0, 1, 1, 0), "identity"),  # one channel, K = 9 (one K-step)
])
def test_conv_stemh_emulated(monkeypatch, shape, pad, layout):
    """The few-channel forward convolution in 2xFP16 (per-tile activation
    scales, per-row filter scales), emulated, within 1e-5 normwise of the
    oracle; with GFB_CONV_F16=0 the TF32 stem kernel runs instead."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import abi
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_STEMH_ALL", "1")
    N, C, K, H, W, R, S = shape
    fn = _conv_graph("fwd", N, C, K, H, W, R, S, (1, 1), pad)
    lay = [(0, 2, 3, 1), None] if layout == "nhwc" else None
    h = host_compile(fn, optimize=False, conv_layout=layout, parameter_layouts=lay)
    kinds = [L.kind for L in h.lowered.launches]
    assert {abi.K_CONV_STEMH, abi.K_CONV_STEMH_C3R7} & set(kinds) and abi.K_SPLIT_TF32 not in kinds, \
        [L.label for L in h.lowered.launches]
    if (C, R, S) == (3, 7, 7):
        assert abi.K_CONV_STEMH_C3R7 in kinds
    rng = np.random.default_rng(17)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0][:, :, : H // 2] *= 1e-3  # tiles of different magnitude: the per-tile scales differ
    tens = [gf.tensor_from_flat(gf.ElementType.F32, v.shape, v, h.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = emulate(h, tens)[0]
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5
    monkeypatch.setenv("GFB_CONV_F16", "0")
    h2 = host_compile(fn, optimize=False, conv_layout=layout, parameter_layouts=lay)
    assert not {abi.K_CONV_STEMH, abi.K_CONV_STEMH_C3R7} & {L.kind for L in h2.lowered.launches}


@pytest.mark.parametrize("layout,fallback", [("identity", False), ("nhwc", False), ("nhwc", True)])
def test_stem_relu_side_output_emulated(monkeypatch, layout, fallback):
    """Relu(Conv2D) of the 3-channel 7x7 stem: the stem kernel writes Relu(y)
    beside y (gfb_stemh_args.flags bit 0) and no Relu map is launched; both
    results within 1e-5 of the oracle, the Relu exactly Relu of the conv.
    With the stem kernels off (GFB_CONV_STEM=0) the planned Relu is emitted
    as a map after the conv's other kernel."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import abi
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    if fallback:
        monkeypatch.setenv("GFB_CONV_STEM", "0")
    Ko, F32 = gf.OpKind, gf.ElementType.F32
    fn = gf.Function("stem_relu")
    x = fn.add_parameter(F32, (2, 3, 12, 40))
    w = fn.add_parameter(F32, (64, 3, 7, 7))
    c = fn.add_node(Ko.CONV2D, [x, w], {"strides": (1, 1), "padding": (3, 3, 3, 3)})
    r = fn.add_node(Ko.RELU, [c])
    # y and Relu(y) stay materialised intermediates (two readers each, as in config D)
    fn.set_results([fn.add_node(Ko.NEGATE, [c]), fn.add_node(Ko.NEGATE, [r]),
                    fn.add_node(Ko.MULTIPLY, [c, r]), fn.add_node(Ko.SUM, [r], {"reduction_axes": (1,)})])
    h = host_compile(fn, optimize=False, conv_layout=layout)
    stem = [L for L in h.lowered.launches if L.kind in (abi.K_CONV_STEMH, abi.K_CONV_STEMH_C3R7)]
    relu_maps = [L for L in h.lowered.launches if "map:Relu" in L.label]
    if fallback:
        assert not stem and len(relu_maps) == 1, [L.label for L in h.lowered.launches]
    else:
        assert stem and stem[0].args.flags == 1 and not relu_maps, [L.label for L in h.lowered.launches]
    rng = np.random.default_rng(29)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(F32, v.shape, v, h.parameter_signature[i][1]) for i, v in enumerate(ins)]
    got = emulate(h, tens)
    ref = interp.run_function(fn, ins)
    assert G.normwise(got[0], ref[0]) <= 1e-5
    # -Relu(y) from -y: y > 0 -> -y, else -0
    assert G.same_bits(got[1], np.where(got[0] < 0, got[0], np.float32(-0.0)).astype(np.float32))


@pytest.mark.parametrize("shape,pad,xlay", [
    ((2, 3, 64, 12, 40, 7, 7), (3, 3, 3, 3), "identity"),  # the stem's shapes: NCHW image, channel-last dy
    ((3, 3, 64, 9, 33, 7, 7), (2, 4, 3, 1), "nhwc"),       # partial 2 x 32 tiles, asymmetric padding
])
def test_conv_stemwh_emulated(monkeypatch, shape, pad, xlay):
    """The 3-channel 7x7 weight gradient on gfb_conv_stemwh_kernel (per-CTA
    partials over contiguous pixel-tile ranges + the ordered reduction),
    emulated, within 1e-5 normwise of the oracle."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import abi
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    N, C, K, H, W, R, S = shape
    fn = _conv_graph("wgrad", N, C, K, H, W, R, S, (1, 1), pad)
    nhwc = (0, 2, 3, 1)
    h = host_compile(fn, optimize=False, parameter_layouts=[nhwc if xlay == "nhwc" else None, None, nhwc])
    kinds = [L.kind for L in h.lowered.launches]
    assert abi.K_CONV_STEMWH_C3R7 in kinds, [L.label for L in h.lowered.launches]
    assert any(":splitk" in L.label for L in h.lowered.launches)
    rng = np.random.default_rng(23)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(gf.ElementType.F32, v.shape, v, h.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = emulate(h, tens)[0]
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("op,shape,stride,pad", [
    ("fwd", (2, 32, 64, 8, 9, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (2, 64, 96, 9, 9, 3, 3), (2, 2), (1, 1, 1, 1)),
    ("fwd", (1, 32, 64, 7, 7, 1, 1), (2, 2), (0, 0, 0, 0)),
    ("dgrad", (2, 40, 64, 8, 7, 3, 3), (1, 1), (1, 0, 0, 1)),
    ("dgrad", (2, 16, 128, 6, 6, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (2, 12, 40, 9, 8, 3, 3), (2, 1), (0, 1, 1, 0)),    # 4-channel pieces, K-blocks span taps
    ("fwd", (2, 3, 64, 12, 11, 7, 7), (1, 1), (3, 3, 3, 3)),   # 3 channels: zero-padded copies
])
def test_conv_fused_gather_emulated(monkeypatch, op, shape, stride, pad):
    """NHWC convolutions whose gathered channels come in 16-byte pieces take
    gfb_conv_tcg_kernel (gather + split inside the GEMM): no im2col planes.
    A 3-channel input is zero-padded to 4 channels first (GFB_PAD_CHANNELS_FWD,
    with the patch-staged stem kernel off)."""
    monkeypatch.setenv("GFB_PAD_CHANNELS_FWD", "1")
    monkeypatch.setenv("GFB_CONV_STEM", "0")
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import abi
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_CONV_F16", "0")
    N, C, K, H, W, R, S = shape
    fn = _conv_graph(op, N, C, K, H, W, R, S, stride, pad)
    nhwc = (0, 2, 3, 1)
    h = host_compile(fn, optimize=False, conv_layout="nhwc", parameter_layouts=[nhwc, None, nhwc][: len(fn.parameters)])
    kinds = [L.kind for L in h.lowered.launches]
    assert set(kinds) & {abi.K_CONV_TCG64, abi.K_CONV_TCG128, abi.K_CONV_TCX64, abi.K_CONV_TCX128}, \
        [L.label for L in h.lowered.launches]
    assert not any(L.label.startswith("split_a") for L in h.lowered.launches)
    rng = np.random.default_rng(9)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(gf.ElementType.F32, v.shape, v, h.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = emulate(h, tens)[0]
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


@pytest.mark.parametrize("op,shape,stride,pad", [
    ("fwd", (2, 32, 64, 8, 9, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (3, 64, 96, 9, 9, 3, 3), (2, 2), (1, 1, 1, 1)),
    ("fwd", (2, 32, 64, 7, 7, 1, 1), (2, 2), (0, 0, 0, 0)),
    ("fwd", (1, 32, 128, 20, 3, 3, 3), (1, 2), (1, 1, 1, 1)),
    ("dgrad", (2, 40, 64, 8, 7, 3, 3), (1, 1), (1, 0, 0, 1)),
])
def test_conv_tma_box_emulated(monkeypatch, op, shape, stride, pad):
    """An intermediate activation (arena) feeding an NHWC convolution takes
    gfb_conv_tcx_kernel: A tiles are TMA boxes of output pixels."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import abi
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_CONV_F16", "0")
    Ko, F32 = gf.OpKind, gf.ElementType.F32
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
    h = host_compile(fn, optimize=False, conv_layout="nhwc")
    kinds = [L.kind for L in h.lowered.launches]
    assert set(kinds) & {abi.K_CONV_TCX64, abi.K_CONV_TCX128}, [L.label for L in h.lowered.launches]
    rng = np.random.default_rng(13)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(F32, v.shape, v) for v in ins]
    out = emulate(h, tens)[0]
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


def test_resnet_nhwc_layout_assignment_emulated():
    """Config D at reduced size under conv_layout='nhwc': conversions are
    inserted by layout assignment and fused away as index maps."""
    case = next(c for c in G.load("workloads.json.gz") if c["name"] == "resnet_D_small")
    fn = G.fn_of(case["fn"])
    ident = host_compile(fn)
    nhwc = host_compile(fn, conv_layout="nhwc")
    assert sum(1 for n in nhwc.graph.nodes.values() if n.op.value == "ConvertLayout") > 0
    # ConvertLayout costs no launch of its own; channel-last storage may keep
    # a pool-window Reshape materialised that the identity plan reads as a view
    assert len(nhwc.lowered.launches) <= len(ident.lowered.launches) + 4
    # the pool composite's flattened window matrices are stored channel-last
    # (sub-axis storage) and its one-hot selections share one launch
    assert any(b.subaxes for b in nhwc.lowered.buffers.values())
    assert any("+" in L.label for L in nhwc.lowered.launches)
    _compare(emulate(nhwc, [G.tensor_of(d) for d in case["inputs"]]), case["outputs"], "resnet nhwc")


@pytest.mark.parametrize("m,k,n,et", [(2, 2, 2, "F64"), (1, 4, 9, "F32"), (4, 1, 7, "F32"), (2, 0, 3, "F64"), (3, 3, 5, "F64")])
def test_tiny_dot_fused_bit_exact(m, k, n, et):
    """Dots with k <= 4 lower to VM multiply-add chains (no Dot launch) and
    keep the reference order bit for bit, NaN/inf/-0 included."""
    import paper_1801_08058_b200 as gf
    from oracle import interp

    et = getattr(gf.ElementType, et)
    fn = gf.Function("tiny")
    a = fn.add_parameter(et, (m, k))
    b = fn.add_parameter(et, (k, n))
    fn.set_results([fn.add_node(gf.OpKind.RELU, [fn.add_node(gf.OpKind.DOT, [a, b])])])
    h = host_compile(fn, optimize=False)
    assert all(L.label.startswith("map:") for L in h.lowered.launches), [L.label for L in h.lowered.launches]
    rng = np.random.default_rng(m * 10 + k)
    A = rng.uniform(-1, 1, size=(m, k)).astype(et.numpy_dtype)
    B = rng.uniform(-1, 1, size=(k, n)).astype(et.numpy_dtype)
    if A.size:
        A.reshape(-1)[0] = -0.0
    if B.size > 2:
        B.reshape(-1)[1] = np.inf
        B.reshape(-1)[2] = np.nan
    out = emulate(h, [gf.tensor_from_flat(et, A.shape, A), gf.tensor_from_flat(et, B.shape, B)])[0]
    assert G.same_bits(out, interp.run_function(fn, [A, B])[0])


@pytest.mark.parametrize("mn", [True, False])
@pytest.mark.parametrize("shape,pad", [((2, 32, 16, 9, 8, 3, 3), (1, 1, 1, 1)), ((2, 5, 8, 7, 7, 3, 3), (1, 0, 0, 1)),
                                       ((3, 12, 132, 6, 5, 3, 3), (1, 1, 0, 2)), ((2, 3, 64, 12, 11, 7, 7), (3, 3, 3, 3))])
def test_wgrad_channel_last_rows_emulated(monkeypatch, shape, pad, mn):
    """ConvBackpropFilter over channel-last data: the MN-major kernel
    (gfb_tcgw_args: 16-byte loads of x and dy, split in the kernel) when the
    channel counts are multiples of 4, else rows (r, s, c) on the element
    gather so lanes read contiguous channels (gfb_tcgg_args.pad0 == 1)."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import abi
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    monkeypatch.setenv("GFB_CONV_F16", "0")  # (the 3-channel 7x7 case would take the 2xFP16 stem kernel)
    monkeypatch.setenv("GFB_TCGW", "1" if mn else "0")
    N, C, K, H, W, R, S = shape
    fn = _conv_graph("wgrad", N, C, K, H, W, R, S, (1, 1), pad)
    nhwc = (0, 2, 3, 1)
    h = host_compile(fn, optimize=False, conv_layout="nhwc", parameter_layouts=[nhwc, None, nhwc])
    labels = [L.label for L in h.lowered.launches]
    if mn and K % 4 == 0 and (C % 4 == 0 or C < 32):  # few channels: zero-padded copy of x
        assert any(L.kind in (abi.K_CONV_TCGW64, abi.K_CONV_TCGW128) for L in h.lowered.launches), labels
        assert not any(L.kind == abi.K_SPLIT_TF32 for L in h.lowered.launches), labels  # no dy planes
    else:
        tg = [L for L in h.lowered.launches if L.kind in (abi.K_CONV_TCGG64, abi.K_CONV_TCGG128)]
        assert tg and tg[0].args.pad0 == 1, labels
    rng = np.random.default_rng(21)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    tens = [gf.tensor_from_flat(gf.ElementType.F32, v.shape, v, h.parameter_signature[i][1]) for i, v in enumerate(ins)]
    out = emulate(h, tens)[0]
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-5


def test_input_row_chunks_emulated(monkeypatch):
    """A large caller input is split and multiplied in row chunks (so its
    H2D copy pipelines with the first GEMM): every result bit-identical to
    the unchunked plan, the chunk launches read disjoint input pieces, and
    the first GEMM chunk depends only on its own split chunk."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import schedule
    from paper_1801_08058_b200 import workloads as W

    st = W.mlp_step(gf, batch=2048, in_dim=256, hidden=(256,), out_dim=256)
    ins = W.step_inputs(st, W.parameter_shapes(st), seed=5)
    tens = [gf.tensor_from_flat(gf.ElementType.F32, v.shape, v) for v in ins]
    monkeypatch.setenv("GFB_INPUT_CHUNK_MIN_MB", "1")
    monkeypatch.setenv("GFB_INPUT_CHUNKS", "4")
    h = host_compile(st.fn)
    labels = [L.label for L in h.lowered.launches]
    assert sum(lb.startswith("split16#") and ":rows" in lb for lb in labels) == 4, labels
    # both layers follow the input's row chunks, in chunk-major order
    assert sum(lb.startswith("dot_f16#") and ":rows" in lb for lb in labels) == 8, labels
    chunked = [lb for lb in labels if ":rows" in lb]
    assert [lb.split(":rows")[1].split(":")[0] for lb in chunked] == [r for r in ("0", "512", "1024", "1536") for _ in range(3)]
    chunked = emulate(h, tens)
    monkeypatch.setenv("GFB_INPUT_CHUNKS", "1")
    plain = emulate(host_compile(st.fn), tens)
    for a, b in zip(chunked, plain):
        assert G.same_bits(a, b)
    # input pieces: x in 4 row pieces, each split chunk reads exactly one
    in_bytes = [v.nbytes for v in ins]
    p_in, p_off, p_len, off, reads = schedule.io_pieces(h.lowered, in_bytes)
    xs = [p for p in range(len(p_in)) if p_in[p] == 0]
    assert len(xs) == 4 and sum(p_len[p] for p in xs) == ins[0].nbytes
    splits = [i for i, L in enumerate(h.lowered.launches) if L.label.startswith("split16#") and ":rows" in L.label]
    assert [reads[off[i]:off[i + 1]] for i in splits] == [[p] for p in xs]
    # the schedule lets GEMM chunk 0 wait for split chunk 0 only (not the later chunks)
    stream_of, doff, deps = schedule.build(h.lowered)
    g0 = next(i for i, L in enumerate(h.lowered.launches) if L.label.startswith("dot_f16#") and ":rows0" in L.label)
    assert not set(deps[doff[g0]:doff[g0 + 1]]) & set(splits[1:])


def _conv_fn(gf, op, shape, stride, pad):
    Ko, F32 = gf.OpKind, gf.ElementType.F32
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
    return fn


@pytest.mark.parametrize("op,shape,stride,pad", [
    ("fwd", (2, 64, 64, 8, 9, 3, 3), (1, 1), (1, 1, 1, 1)),
    ("fwd", (3, 64, 96, 9, 9, 3, 3), (2, 2), (1, 1, 1, 1)),
    ("fwd", (2, 128, 200, 7, 7, 1, 1), (2, 2), (0, 0, 0, 0)),
    ("dgrad", (2, 40, 64, 8, 7, 3, 3), (1, 1), (1, 0, 0, 1)),
])
def test_conv_tcxh_emulated(monkeypatch, op, shape, stride, pad):
    """Channel-scaled fp16 activation planes + filter planes divided by the
    same scales (2xFP16 TMA-box convolution), with channels 1e20 apart:
    normwise within 1e-6 of the oracle."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import abi
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    fn = _conv_fn(gf, op, shape, stride, pad)
    h = host_compile(fn, optimize=False, conv_layout="nhwc")
    kinds = [L.kind for L in h.lowered.launches]
    assert {abi.K_CHMAX, abi.K_CHSPLIT, abi.K_FSPLIT} <= set(kinds), [L.label for L in h.lowered.launches]
    assert set(kinds) & {abi.K_CONV_TCXH64, abi.K_CONV_TCXH128}
    rng = np.random.default_rng(17)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0][:, 1] *= np.float32(1e-12)  # one channel far below the others: scales are per channel
    ins[0][:, 2] *= np.float32(1e8)
    tens = [gf.tensor_from_flat(gf.ElementType.F32, v.shape, v) for v in ins]
    out = emulate(h, tens)[0]
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-6


@pytest.mark.parametrize("shape,pad", [((2, 64, 64, 9, 10, 3, 3), (1, 1, 1, 1)), ((3, 128, 64, 7, 7, 1, 1), (0, 0, 0, 0)),
                                       ((2, 64, 128, 8, 8, 3, 3), (1, 0, 0, 1))])
def test_conv_tcgwh_emulated(monkeypatch, shape, pad):
    """2xFP16 weight gradient on the channel-scaled planes of x and dy:
    normwise within 1e-6 of the oracle."""
    import paper_1801_08058_b200 as gf
    from paper_1801_08058_b200 import abi
    from oracle import interp

    monkeypatch.setenv("GFB_CONV", "tc")
    Ko, F32 = gf.OpKind, gf.ElementType.F32
    N, C, K, H, W, R, S = shape
    fn = gf.Function("wgrad")
    x = fn.add_parameter(F32, (N, C, H, W))
    Ho, Wo = H + pad[0] + pad[1] - R + 1, W + pad[2] + pad[3] - S + 1
    d = fn.add_parameter(F32, (N, K, Ho, Wo))
    g = fn.add_node(Ko.CONV_BACKPROP_FILTER, [fn.add_node(Ko.RELU, [x]), fn.add_node(Ko.NEGATE, [d])],
                    {"filter_shape": (K, C, R, S), "padding": pad}, allow_internal=True)
    fn.set_results([g])
    h = host_compile(fn, optimize=False, conv_layout="nhwc")
    kinds = [L.kind for L in h.lowered.launches]
    assert set(kinds) & {abi.K_CONV_TCGWH64, abi.K_CONV_TCGWH128}, [L.label for L in h.lowered.launches]
    rng = np.random.default_rng(23)
    ins = [rng.uniform(-1, 1, size=fn.nodes[p].output.shape).astype(np.float32) for p in fn.parameters]
    ins[0][:, 3] *= np.float32(1e-9)
    tens = [gf.tensor_from_flat(F32, v.shape, v) for v in ins]
    out = emulate(h, tens)[0]
    interp.set_threads(interp.max_threads())
    assert G.normwise(out, interp.run_function(fn, ins)[0]) <= 1e-6
