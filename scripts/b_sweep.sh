#!/bin/bash
# Build scripts/b_sweep (grid-size sweep of config B's generated kernel); run it on the GPU box.
set -e
D=$(mktemp -d)
python - "$D" <<'PY'
import sys
sys.path[:0] = ['.', 'tests']
import paper_1801_08058_b200 as gf
from paper_1801_08058_b200 import workloads as W, jit, abi
from hostcompile import host_compile
d = sys.argv[1]
low = host_compile(W.fused_chain(gf, rows=65536, cols=1024)).lowered
recs, blob = low.pack()
r = recs[0]
src = jit.generate(low.launches[0].kind, abi.EwArgs.from_buffer_copy(blob[r.arg_offset:r.arg_offset + r.arg_size]), r.block[0])[0]
body = src.split("\n", 5)[5]  # drop the includes / macros the harness defines once
variants = {
    "v0": body,
    "v1": body.replace("\nfor (uint32_t rl = ", '\n_Pragma("unroll") for (uint32_t rl = '),
    "v2": body.replace("__launch_bounds__(256, 4)", "__launch_bounds__(256, 6)"),
}
for v, b in variants.items():
    b = b.replace("namespace m0", f"namespace {v}").replace("m0::run", f"{v}::run").replace("gfb_jit_ew", f"k_{v}")
    open(f"{d}/{v}.inc", "w").write(b)
PY
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I"$D" -Ipaper_1801_08058_b200/csrc -Iinclude \
  -o scripts/b_sweep scripts/b_sweep.cu
rm -rf "$D"
