"""Training-step and fused-chain graphs for the BASELINE.json configs.

Every builder takes `api` — any module exposing the reference construction
API (`Function`, `ElementType`, `OpKind`, `build_softmax`, `differentiate`,
`topological_order`) — so the *same* code builds the graph with the
reference package (golden generation, `tests/golden/make_golden.py`) and
with this package (the B200 path).  A training step is one Function, exactly
as SURVEY.md §3.3 describes: loss graph -> `differentiate` -> per-parameter
`Subtract(p, Multiply(Broadcast(lr), grad))`, results = new parameters +
the embedded forward loss.

Configs (BASELINE.json `configs`):
  A  MLP 784-512-10, batch 128                       `mlp_step`
  B  Relu(a + Broadcast(c)) * b and its row Sum        `fused_chain`
  C  small CNN 2xConv + maxpool composite + fc         `cnn_step`
  D  ResNet-18-style convnet, NCHW<->NHWC              `resnet_step`
  E  wide MLP, L layers of width W, global batch       `mlp_step(hidden=[W]*L)`
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class StepGraph:
    fn: object  # api.Function
    param_names: list  # one per parameter of fn, in order
    weight_names: list  # trained parameters (results 0..k-1 are their new values)
    loss_index: int  # position of the loss among the results


def _loss_node_id(api, fn_fwd, loss_id: int) -> int:
    """Id of the forward loss inside the differentiated graph.

    `differentiate` adds the P parameters first, then every non-parameter
    node in topological order (reference `autodiff.py:58-75`), so the copy
    of node n has id P + its rank among those nodes.
    """
    order = [n for n in api.topological_order(fn_fwd) if fn_fwd.nodes[n].op is not api.OpKind.PARAMETER]
    return len(fn_fwd.parameters) + 1 + order.index(loss_id)


def _append_sgd(api, g, wrt_ids_in_g, grad_refs, lr: float, et):
    lr_id = g.add_constant(et, (), [lr])
    new = []
    for pid, grad in zip(wrt_ids_in_g, grad_refs):
        shape = g.nodes[pid].output.shape
        scaled = g.add_node(
            api.OpKind.MULTIPLY,
            [g.add_node(api.OpKind.BROADCAST, [lr_id], {"output_shape": shape, "broadcast_axes": tuple(range(len(shape)))}), grad],
        )
        new.append(g.add_node(api.OpKind.SUBTRACT, [pid, scaled]))
    return new


def _softmax_xent(api, fn, logits, t, batch, et):
    """loss = -sum(t * log softmax(logits)) / batch (batch = the GLOBAL batch
    under data parallelism, so per-rank partial losses and gradients sum)."""
    K = api.OpKind
    p = api.build_softmax(fn, logits, 1)
    tl = fn.add_node(K.MULTIPLY, [t, fn.add_node(K.LOG, [p])])
    s = fn.add_node(K.SUM, [tl], {"reduction_axes": (0, 1)})
    return fn.add_node(K.DIVIDE, [fn.add_node(K.NEGATE, [s]), fn.add_constant(et, (), [float(batch)])])


def _training_step(api, fwd, loss, names, weights, lr, et) -> StepGraph:
    fwd.set_results([loss])
    wrt = [fwd.parameters[names.index(w)] for w in weights]
    g = api.differentiate(fwd, wrt)
    loss_in_g = _loss_node_id(api, fwd, loss)
    grads = list(g.results)
    new = _append_sgd(api, g, [g.parameters[names.index(w)] for w in weights], grads, lr, et)
    g.set_results(new + [loss_in_g])
    return StepGraph(g, names + ["seed"], list(weights), len(new))


def mlp_step(api, batch=128, in_dim=784, hidden=(512,), out_dim=10, lr=0.01, bias=True, f32=True,
             loss_batch=None) -> StepGraph:
    """MLP training step (config A; config E with hidden=[4096]*7, in=out=4096).

    `batch` is the per-replica batch the graph is specialised to;
    `loss_batch` (default `batch`) is the divisor of the summed loss."""
    et = api.ElementType.F32 if f32 else api.ElementType.F64
    K = api.OpKind
    fn = api.Function("mlp_step")
    names = ["x"]
    x = fn.add_parameter(et, (batch, in_dim))
    dims = [in_dim] + list(hidden) + [out_dim]
    layers = []
    for i in range(len(dims) - 1):
        w = fn.add_parameter(et, (dims[i], dims[i + 1]))
        names.append(f"W{i + 1}")
        b = None
        if bias:
            b = fn.add_parameter(et, (dims[i + 1],))
            names.append(f"b{i + 1}")
        layers.append((w, b))
    t = fn.add_parameter(et, (batch, out_dim))
    names.append("t")
    h = x
    for i, (w, b) in enumerate(layers):
        h = fn.add_node(K.DOT, [h, w])
        if b is not None:
            h = fn.add_node(K.ADD, [h, fn.add_node(K.BROADCAST, [b], {"output_shape": (batch, dims[i + 1]), "broadcast_axes": (0,)})])
        if i < len(layers) - 1:
            h = fn.add_node(K.RELU, [h])
    loss = _softmax_xent(api, fn, h, t, loss_batch or batch, et)
    weights = [n for n in names if n[0] in "Wb"]
    return _training_step(api, fn, loss, names, weights, lr, et)


def wide_mlp_step(api, batch=65536, width=4096, layers=8, loss_batch=None, lr=0.01) -> StepGraph:
    """Config E: `layers` Dot+bias layers of width x width with Relu between
    them, softmax cross-entropy over `width` classes, SGD."""
    return mlp_step(api, batch=batch, in_dim=width, hidden=(width,) * (layers - 1), out_dim=width, lr=lr,
                    loss_batch=loss_batch)


def conv_gain_of(workload: str) -> float:
    """Scale of the He-style conv filter bound per config.  Config D (no
    normalisation, 8 residual additions) at gain 1 drives the logits so far
    apart that softmax probabilities underflow to 0 and the reference loss
    t * log(p) becomes 0 * -inf = NaN; at 0.5 the 224x224 step stays finite
    (loss ~2.2, near log 10)."""
    return 0.5 if workload == "D" else 1.0


def x_range_of(workload: str) -> tuple:
    """Input distribution of x per config: U(-1, 1) for
    config E, U(0, 1) (image-like) for the others."""
    return (-1.0, 1.0) if workload == "E" else (0.0, 1.0)


def maxpool2x2(api, fn, x, shape):
    """Differentiable 2x2/2 max-pool composite (SURVEY.md §7 hard part 8)."""
    K = api.OpKind
    et = fn.nodes[x].output.element_type
    n, c, h, w = shape
    h2, w2 = h // 2, w // 2
    m = n * c * h2 * w2
    six = fn.add_node(K.RESHAPE, [x], {"input_order": (0, 1, 2, 3), "output_shape": (n, c, h2, 2, w2, 2)})
    win = fn.add_node(K.RESHAPE, [six], {"input_order": (3, 5, 0, 1, 2, 4), "output_shape": (4, m)})
    rows = []
    for k in range(4):
        sel = fn.add_constant(et, (1, 4), [1.0 if j == k else 0.0 for j in range(4)])
        rows.append(fn.add_node(K.DOT, [sel, win]))
    top = fn.add_node(K.MAXIMUM, [fn.add_node(K.MAXIMUM, [rows[0], rows[1]]), fn.add_node(K.MAXIMUM, [rows[2], rows[3]])])
    return fn.add_node(K.RESHAPE, [top], {"input_order": (0, 1), "output_shape": (n, c, h2, w2)})


def cnn_step(api, batch=256, image=32, channels=(3, 16, 32), classes=10, lr=0.01, f32=True,
             loss_batch=None) -> StepGraph:
    """Small CNN training step (config C): conv-relu-conv-relu-pool-fc-softmax."""
    et = api.ElementType.F32 if f32 else api.ElementType.F64
    K = api.OpKind
    c0, c1, c2 = channels
    fn = api.Function("cnn_step")
    x = fn.add_parameter(et, (batch, c0, image, image))
    k1 = fn.add_parameter(et, (c1, c0, 3, 3))
    k2 = fn.add_parameter(et, (c2, c1, 3, 3))
    feat = c2 * (image // 2) * (image // 2)
    wf = fn.add_parameter(et, (feat, classes))
    t = fn.add_parameter(et, (batch, classes))
    names = ["x", "K1", "K2", "Wf", "t"]
    conv = {"strides": (1, 1), "padding": (1, 1, 1, 1)}
    h = fn.add_node(K.RELU, [fn.add_node(K.CONV2D, [x, k1], conv)])
    h = fn.add_node(K.RELU, [fn.add_node(K.CONV2D, [h, k2], conv)])
    p = maxpool2x2(api, fn, h, (batch, c2, image, image))
    flat = fn.add_node(K.RESHAPE, [p], {"input_order": (0, 1, 2, 3), "output_shape": (batch, feat)})
    logits = fn.add_node(K.DOT, [flat, wf])
    loss = _softmax_xent(api, fn, logits, t, loss_batch or batch, et)
    return _training_step(api, fn, loss, names, ["K1", "K2", "Wf"], lr, et)


def resnet_step(api, batch=128, image=224, widths=(64, 128, 256, 512), blocks=2, classes=10, lr=0.01,
                f32=True, loss_batch=None) -> StepGraph:
    """ResNet-18-style training step (config D).

    The IR has no strided-conv gradient (`autodiff.py:226-230`), no BatchNorm
    and no max-pool op, so:
    * the stem is a 7x7 stride-1 pad-3 conv followed by two pool composites
      (224 -> 56);
    * each stage runs `blocks` BasicBlocks of two 3x3 stride-1 convs;
    * stages are joined by a pool composite and a 1x1 projection shortcut.
    The head is a spatial Sum scaled by 1/(H*W), then fc -> softmax
    cross-entropy.  Compile it with conv_layout="nhwc" for the layout
    assignment the config names."""
    et = api.ElementType.F32 if f32 else api.ElementType.F64
    K = api.OpKind
    fn = api.Function("resnet_step")
    names = ["x"]
    x = fn.add_parameter(et, (batch, 3, image, image))
    pad1 = {"strides": (1, 1), "padding": (1, 1, 1, 1)}
    weights = []

    def param(shape, name):
        pid = fn.add_parameter(et, shape)
        names.append(name)
        weights.append(name)
        return pid

    stem = param((widths[0], 3, 7, 7), "K_stem")
    h = fn.add_node(K.RELU, [fn.add_node(K.CONV2D, [x, stem], {"strides": (1, 1), "padding": (3, 3, 3, 3)})])
    size, ch = image, widths[0]
    for _ in range(2):
        h = maxpool2x2(api, fn, h, (batch, ch, size, size))
        size //= 2
    for si, w in enumerate(widths):
        if si > 0:
            h = maxpool2x2(api, fn, h, (batch, ch, size, size))
            size //= 2
        for bi in range(blocks):
            k1 = param((w, ch, 3, 3), f"K{si}_{bi}a")
            k2 = param((w, w, 3, 3), f"K{si}_{bi}b")
            y = fn.add_node(K.RELU, [fn.add_node(K.CONV2D, [h, k1], pad1)])
            y = fn.add_node(K.CONV2D, [y, k2], pad1)
            if ch != w:
                kp = param((w, ch, 1, 1), f"P{si}_{bi}")
                short = fn.add_node(K.CONV2D, [h, kp], {"strides": (1, 1), "padding": (0, 0, 0, 0)})
            else:
                short = h
            h = fn.add_node(K.RELU, [fn.add_node(K.ADD, [y, short])])
            ch = w
    pooled = fn.add_node(K.SUM, [h], {"reduction_axes": (2, 3)})
    scale = fn.add_constant(et, (), [1.0 / (size * size)])
    pooled = fn.add_node(K.MULTIPLY, [pooled, fn.add_node(K.BROADCAST, [scale], {"output_shape": (batch, ch), "broadcast_axes": (0, 1)})])
    wf = param((ch, classes), "Wf")
    t = fn.add_parameter(et, (batch, classes))
    names.append("t")
    logits = fn.add_node(K.DOT, [pooled, wf])
    loss = _softmax_xent(api, fn, logits, t, loss_batch or batch, et)
    return _training_step(api, fn, loss, names, weights, lr, et)


def fused_chain(api, rows=65536, cols=1024, f32=True):
    """Config B: t3 = Relu(a + Broadcast(c)) * b; results t3 and Sum_axis1(t3)."""
    et = api.ElementType.F32 if f32 else api.ElementType.F64
    K = api.OpKind
    fn = api.Function("fused_chain")
    a = fn.add_parameter(et, (rows, cols))
    b = fn.add_parameter(et, (rows, cols))
    c = fn.add_parameter(et, (cols,))
    t1 = fn.add_node(K.ADD, [a, fn.add_node(K.BROADCAST, [c], {"output_shape": (rows, cols), "broadcast_axes": (0,)})])
    t3 = fn.add_node(K.MULTIPLY, [fn.add_node(K.RELU, [t1]), b])
    fn.set_results([t3, fn.add_node(K.SUM, [t3], {"reduction_axes": (1,)})])
    return fn


# ---------------------------------------------------------------------------
# Synthetic inputs (seeded, identical on every backend)


def _uniform(rng, shape, lo, hi, dtype):
    return rng.uniform(lo, hi, size=shape).astype(dtype)


def _one_hot(rng, batch, classes, dtype):
    t = np.zeros((batch, classes), dtype=dtype)
    t[np.arange(batch), rng.integers(0, classes, size=batch)] = 1.0
    return t


def step_inputs(step: StepGraph, fn_shapes: dict, seed=0, f32=True, x_range=(0.0, 1.0), conv_gain=1.0) -> list:
    """Arrays for every parameter of a training step, in parameter order."""
    dtype = np.float32 if f32 else np.float64
    rng = np.random.default_rng(seed)
    out = []
    for name in step.param_names:
        shape = fn_shapes[name]
        if name == "x":
            out.append(_uniform(rng, shape, x_range[0], x_range[1], dtype))
        elif name == "t":
            out.append(_one_hot(rng, shape[0], shape[1], dtype))
        elif name == "seed":
            out.append(np.ones(shape, dtype=dtype))
        elif len(shape) == 4:  # conv filter [K, C, R, S]: He-style fan-in bound
            bound = conv_gain * float(np.sqrt(6.0 / (shape[1] * shape[2] * shape[3])))
            out.append(_uniform(rng, shape, -bound, bound, dtype))
        else:
            fan = shape[0] if len(shape) >= 2 else 10
            bound = 0.1 if fan <= 1024 else 1.0 / 64.0
            out.append(_uniform(rng, shape, -bound, bound, dtype))
    return out


def parameter_shapes(step: StepGraph) -> dict:
    g = step.fn
    return {name: tuple(g.nodes[pid].output.shape) for name, pid in zip(step.param_names, g.parameters)}


def chain_inputs(rows, cols, seed=1, f32=True) -> list:
    dtype = np.float32 if f32 else np.float64
    rng = np.random.default_rng(seed)
    return [_uniform(rng, (rows, cols), -1, 1, dtype), _uniform(rng, (rows, cols), -1, 1, dtype), _uniform(rng, (cols,), -1, 1, dtype)]
