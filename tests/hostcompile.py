"""Host-side compile with the oracle as fold evaluator (CPU tests only)."""

from oracle import interp
from paper_1801_08058_b200.layout import Layout
from paper_1801_08058_b200.runtime import prepare_function

import plan_emulator


def host_compile(fn, optimize=True, conv_layout="identity", parameter_layouts=None, private=False, data_parallel=None):
    layouts = None
    if parameter_layouts is not None:
        layouts = [None if o is None else Layout(tuple(o)) for o in parameter_layouts]
    return prepare_function(fn, optimize=optimize, conv_layout=conv_layout, parameter_layouts=layouts,
                            evaluate=interp.fold_evaluator, private=private, data_parallel=data_parallel)


def emulate(h, tensors):
    """Run a HostCompiled plan on the numpy emulator; returns logical arrays."""
    import numpy as np

    from paper_1801_08058_b200.tensor import storage_to_logical

    specs = [(d.element_type.numpy_dtype, d.element_count) for d, _ in h.result_signature]
    outs = plan_emulator.execute(h.lowered, [t.buffer for t in tensors], specs)
    res = []
    for (d, lay), o in zip(h.result_signature, outs):
        res.append(storage_to_logical(o.view(d.element_type.numpy_dtype), d.shape, lay) if d.shape else o.reshape(()))
    return res
