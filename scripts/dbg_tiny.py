import numpy as np, sys
sys.path.insert(0, '.')
import paper_1801_08058_b200 as gf
K = gf.OpKind
for et in (gf.ElementType.F64, gf.ElementType.F32):
    for (m, k, n) in ((2, 2, 2), (1, 4, 8), (4, 1, 16), (3, 3, 300)):
        fn = gf.Function("d"); a = fn.add_parameter(et, (m, k)); b = fn.add_parameter(et, (k, n))
        fn.set_results([fn.add_node(K.DOT, [a, b])])
        exe = gf.compile_function(fn, optimize=False)
        A = np.arange(1, m * k + 1, dtype=et.numpy_dtype).reshape(m, k); B = np.arange(5, 5 + k * n, dtype=et.numpy_dtype).reshape(k, n)
        out = gf.call(exe, [gf.tensor_from_flat(et, (m, k), A), gf.tensor_from_flat(et, (k, n), B)])[0].to_numpy()
        print(et, m, k, n, [L.label for L in exe.lowered.launches], np.array_equal(out, A @ B), out.reshape(-1)[:4], (A @ B).reshape(-1)[:4])
