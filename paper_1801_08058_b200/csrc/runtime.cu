// Executor behind the C ABI in include/gfb200.h.
//
// An executable owns: one device arena (the liveness-planned buffers of all
// fused launches), the constant pool (uploaded once), a device pointer table
// that kernels resolve tensor slots through, and a CUDA graph of the launch
// list captured on the first run.  A run is: write this call's input/output
// pointers into the table (one 8*(2+n_in+n_out)-byte H2D copy) and launch
// the graph — the reference's per-instruction Python dispatch
// (interpreter.py:208-230) becomes a single cudaGraphLaunch.

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gfb200.h"
#include <nvtx3/nvToolsExt.h>

extern "C" const void* gfb_ew_kernel_ptr(int kind);
extern "C" const void* gfb_simt_kernel_ptr(int kind);
extern "C" const void* gfb_tc_kernel_ptr(int kind);
extern "C" const void* gfb_f16_kernel_ptr(int kind);
extern "C" const void* gfb_conv_f16_kernel_ptr(int kind);

namespace {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)f;
    }
    return fn;
}

// K-major fp32 plane [rows, kp] -> 128B-swizzled boxes of 32 (K) x box_rows.
bool encode_plane_map(void* gaddr, int64_t rows, int64_t kp, uint32_t box_rows, void* out) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    alignas(64) CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kp * 4};
    cuuint32_t box[2] = {32, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, gaddr, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out, &map, sizeof(map));
    return true;
}
// MN-major operand (element (mn, k) at k * ld + mn): 3-D view (32 MN, K,
// MN / 32) whose box (32, 32, 4) lands as four 4 KB MN atoms in the
// SWIZZLE_128B_BASE32B layout tcgen05 reads MN-major tf32 operands in
// (SWIZZLE_128B_ATOM_32B; scripts/tma_mn_probe.cu checks it against a host
// product, profiles/r02_tma_mn_probe.txt).
bool encode_mn_map(void* gaddr, int64_t mn, int64_t k, int64_t ld, void* out) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || mn % 32) return false;
    alignas(64) CUtensorMap map;
    cuuint64_t dims[3] = {32, (cuuint64_t)k, (cuuint64_t)(mn / 32)};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, 128};
    cuuint32_t box[3] = {32, 32, 4};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, gaddr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out, &map, sizeof(map));
    return true;
}
// fp16 planes of the 2xFP16 GEMM (gemm_f16.cu).  K-major [rows, kp]:
// 128B-swizzled boxes of 64 (K) x 128 rows.  MN-major (element (mn, k) at
// k * ld + mn, mn % 64 == 0): 3-D view (64 MN, K, MN / 64) with (64, 64, 2)
// boxes, i.e. two 8 KB chunks of 64 K rows x 128 B in the canonical
// SWIZZLE_128B MN-major layout.
bool encode_plane16_map(void* gaddr, int64_t rows, int64_t kp, void* out, uint32_t box_rows = 128) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || kp % 8) return false;
    alignas(64) CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kp * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, gaddr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out, &map, sizeof(map));
    return true;
}
bool encode_mn16_map(void* gaddr, int64_t mn, int64_t k, int64_t ld, void* out) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || mn % 64 || ld % 8) return false;
    alignas(64) CUtensorMap map;
    cuuint64_t dims[3] = {64, (cuuint64_t)k, (cuuint64_t)(mn / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 2, 128};
    cuuint32_t box[3] = {64, 64, 2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, gaddr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out, &map, sizeof(map));
    return true;
}
// Channel-last fp16 activation plane (C, W, H, N innermost first): boxes of
// 64 channels (128 B rows) x bw x bh x bn, traversal strides (1, sx, sy, 1).
bool encode_act16_map(void* gaddr, const int64_t* dims, const int64_t* estrides, uint32_t bw, uint32_t bh, uint32_t bn,
                      uint32_t sx, uint32_t sy, void* out) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    alignas(64) CUtensorMap map;
    cuuint64_t d[4] = {(cuuint64_t)dims[0], (cuuint64_t)dims[1], (cuuint64_t)dims[2], (cuuint64_t)dims[3]};
    cuuint64_t st[3] = {(cuuint64_t)estrides[1] * 2, (cuuint64_t)estrides[2] * 2, (cuuint64_t)estrides[3] * 2};
    cuuint32_t box[4] = {64, bw, bh, bn};
    cuuint32_t es[4] = {1, sx, sy, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, gaddr, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out, &map, sizeof(map));
    return true;
}
// Channel-last 4-D activation (C, W, H, N innermost first) -> boxes of
// 32 channels x bw x bh x bn with traversal strides (1, sx, sy, 1); taps
// outside the tensor read as zero (the convolution's padding).
bool encode_act_map(void* gaddr, const int64_t* dims, const int64_t* estrides, uint32_t bw, uint32_t bh, uint32_t bn,
                    uint32_t sx, uint32_t sy, void* out) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    alignas(64) CUtensorMap map;
    cuuint64_t d[4] = {(cuuint64_t)dims[0], (cuuint64_t)dims[1], (cuuint64_t)dims[2], (cuuint64_t)dims[3]};
    cuuint64_t st[3] = {(cuuint64_t)estrides[1] * 4, (cuuint64_t)estrides[2] * 4, (cuuint64_t)estrides[3] * 4};
    cuuint32_t box[4] = {32, bw, bh, bn};
    cuuint32_t es[4] = {1, sx, sy, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, gaddr, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    std::memcpy(out, &map, sizeof(map));
    return true;
}
}  // namespace

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(GFB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
    } while (0)

// ---- NCCL, loaded on demand so the library has no hard NCCL dependency ----
typedef int ncclResult_t;
typedef void* ncclComm_t;
struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(void*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, char[128], int) = nullptr;  // id passed by value in C
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommRegister)(ncclComm_t, void*, size_t, void**) = nullptr;  // NCCL >= 2.19, optional
    ncclResult_t (*CommDeregister)(ncclComm_t, void*) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

struct NcclUniqueId {
    char internal[128];
};
typedef ncclResult_t (*InitRankFn)(ncclComm_t*, int, NcclUniqueId, int);

int load_nccl() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.loaded) return GFB_OK;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names)
        if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return fail(GFB_ERR_NCCL, std::string("cannot dlopen libnccl.so.2: ") + dlerror());
    g_nccl.GetUniqueId = (ncclResult_t(*)(void*))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.CommRegister = (decltype(g_nccl.CommRegister))dlsym(h, "ncclCommRegister");
    g_nccl.CommDeregister = (decltype(g_nccl.CommDeregister))dlsym(h, "ncclCommDeregister");
    if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy)
        return fail(GFB_ERR_NCCL, "libnccl is missing required symbols");
    g_nccl.loaded = true;
    return GFB_OK;
}

int nccl_fail(ncclResult_t r, const char* what) {
    std::string msg = std::string(what) + " failed: ";
    msg += g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : std::to_string(r);
    return fail(GFB_ERR_NCCL, msg);
}

}  // namespace

struct gfb_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
};

struct gfb_exe {
    int device = 0;
    void* arena = nullptr;
    void* consts = nullptr;
    void** dtab = nullptr;  // device pointer table
    void** htab = nullptr;  // pinned staging copy of the table
    cudaEvent_t tab_done = nullptr;
    // completion of the previous run: the next run (on any stream) waits for
    // it before rewriting the pointer table or touching the arena, so runs
    // of one executable never overlap on the device
    cudaEvent_t run_done = nullptr;
    bool ran = false;
    void* nccl_reg = nullptr;  // ncclCommRegister handle of the arena (GFB_NCCL_REGISTER=1)
    uint32_t n_in = 0, n_out = 0, n_slots = 0;
    std::vector<gfb_launch> launches;
    std::vector<const void*> fns;
    std::vector<unsigned char> args;  // argument blocks, tab pointers patched in
    bool use_graph = false;
    cudaGraphExec_t graph = nullptr;
    cudaStream_t capture_stream = nullptr;
    gfb_comm* comm = nullptr;
    std::mutex mu;
    // multi-stream capture schedule (gfb_exe_set_schedule): stream of each
    // launch and the earlier launches it must wait for (CSR)
    uint32_t n_streams = 1;
    std::vector<uint32_t> stream_of, dep_off, deps;
    std::vector<cudaStream_t> streams;  // streams[0] is capture_stream
    std::vector<cudaEvent_t> done;
    cudaEvent_t fork = nullptr;
    std::vector<cudaEvent_t> joins;
    // host-buffer runs (gfb_exe_set_io / gfb_exe_run_host): device staging
    // buffers of the inputs and results, the inputs each launch reads (CSR)
    // and the last launch writing each result; a second CUDA graph holds the
    // H2D / D2H copies next to the launches
    bool io_set = false;
    std::vector<uint64_t> in_bytes, out_bytes;
    std::vector<void*> dev_in, dev_out;
    std::vector<uint32_t> rd_off, rd, out_writer, in_order;  // rd / in_order: input pieces
    std::vector<uint32_t> pc_in;                             // piece -> input
    std::vector<uint64_t> pc_off, pc_len;                    // piece bytes within its input
    cudaGraph_t hgraph = nullptr;
    cudaGraphExec_t hexec = nullptr;
    std::vector<cudaGraphNode_t> h2d_node, d2h_node;
    std::vector<const void*> cur_hin;
    std::vector<void*> cur_hout;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> in_ev, wr_ev;
    cudaEvent_t io_fork = nullptr, h2d_join = nullptr, d2h_join = nullptr;
};

namespace {

const void* kernel_for(uint32_t kind) {
    if ((kind >= GFB_K_EW_F32 && kind <= GFB_K_EW1_F64) || kind == GFB_K_ROWJIT) return gfb_ew_kernel_ptr((int)kind);
    if (kind == GFB_K_DOT_F32 || kind == GFB_K_DOT_F64 || kind == GFB_K_CONV_F32 || kind == GFB_K_CONV_F64 ||
        kind == GFB_K_DOT_SM_F32 || kind == GFB_K_DOT_SM_F64 || kind == GFB_K_DOT_TH_F32 || kind == GFB_K_DOT_TH_F64)
        return gfb_simt_kernel_ptr((int)kind);
    if (kind == GFB_K_DOT_TC32 || kind == GFB_K_DOT_TC32W || kind == GFB_K_DOT_TC32P || kind == GFB_K_SPLIT_TF32 || kind == GFB_K_CONV_TCG64 ||
        kind == GFB_K_CONV_TCG128 || kind == GFB_K_CONV_TCX64 || kind == GFB_K_CONV_TCX128 || kind == GFB_K_CONV_TCGG64 ||
        kind == GFB_K_CONV_TCGG128 || kind == GFB_K_CONV_TCGW64 || kind == GFB_K_CONV_TCGW128 || kind == GFB_K_CONV_STEM64)
        return gfb_tc_kernel_ptr((int)kind);
    if (kind == GFB_K_DOT_F16P || kind == GFB_K_SPLIT_F16) return gfb_f16_kernel_ptr((int)kind);
    if ((kind >= GFB_K_CHMAX && kind <= GFB_K_CONV_TCGWH128) || kind == GFB_K_CONV_STEMH || kind == GFB_K_CONV_STEMH_C3R7 ||
        kind == GFB_K_CONV_STEMWH_C3R7)
        return gfb_conv_f16_kernel_ptr((int)kind);
    return nullptr;
}

int launch_one(gfb_exe* e, size_t i, cudaStream_t s) {
    const gfb_launch& L = e->launches[i];
    void* blob = e->args.data() + L.arg_offset;
    if (L.kind == GFB_K_ALLREDUCE) {
        const gfb_allreduce_args* a = (const gfb_allreduce_args*)blob;
        if (!e->comm) return fail(GFB_ERR_INVALID, "plan has an all-reduce but no communicator");
        void* ptr = (char*)((a->buf >> 56) == GFB_SLOT_ARENA ? e->arena : nullptr) + (a->buf & ((1ull << 56) - 1));
        if ((a->buf >> 56) != GFB_SLOT_ARENA) return fail(GFB_ERR_INVALID, "all-reduce bucket must live in the arena");
        ncclResult_t r = g_nccl.AllReduce(ptr, ptr, (size_t)a->count, a->dtype == 0 ? 7 /*ncclFloat32*/ : 8 /*ncclFloat64*/,
                                          a->op == 1 ? 2 /*ncclMax*/ : 0 /*ncclSum*/, e->comm->comm, s);
        if (r != 0) return nccl_fail(r, "ncclAllReduce");
        return GFB_OK;
    }
    if (L.kind == GFB_K_MEMSET) {
        const gfb_memset_args* a = (const gfb_memset_args*)blob;
        if ((a->buf >> 56) != GFB_SLOT_ARENA) return fail(GFB_ERR_INVALID, "memset target must live in the arena");
        CUDA_TRY(cudaMemsetAsync((char*)e->arena + (a->buf & ((1ull << 56) - 1)), 0, (size_t)a->bytes, s));
        return GFB_OK;
    }
    if (!e->fns[i]) return GFB_OK;  // folded into a preceding merged kernel (gfb_exe_set_kernel with NULL)
    void* kargs[1] = {blob};
    dim3 grid(L.grid[0], L.grid[1], L.grid[2]), block(L.block[0], L.block[1], L.block[2]);
    cudaError_t err = cudaLaunchKernel(e->fns[i], grid, block, kargs, L.smem, s);
    if (err != cudaSuccess)
        return fail(GFB_ERR_CUDA, std::string("launch ") + std::to_string(i) + " (kind " + std::to_string(L.kind) +
                                      "): " + cudaGetErrorString(err));
    return GFB_OK;
}

int launch_all(gfb_exe* e, cudaStream_t s) {
    for (size_t i = 0; i < e->launches.size(); ++i) {
        int rc = launch_one(e, i, s);
        if (rc != GFB_OK) return rc;
    }
    return GFB_OK;
}

// Capture-time launch order over several streams: every launch waits (by
// event) only for the earlier launches it conflicts with, so independent
// branches of the step (weight gradients next to data gradients, bias sums,
// optimizer updates) become concurrent nodes of the CUDA graph.
int launch_all_streams(gfb_exe* e, cudaStream_t s0) {
    CUDA_TRY(cudaEventRecord(e->fork, s0));
    for (uint32_t k = 1; k < e->n_streams; ++k) CUDA_TRY(cudaStreamWaitEvent(e->streams[k], e->fork, 0));
    for (size_t i = 0; i < e->launches.size(); ++i) {
        const uint32_t sk = e->stream_of[i];
        cudaStream_t st = sk == 0 ? s0 : e->streams[sk];
        for (uint32_t d = e->dep_off[i]; d < e->dep_off[i + 1]; ++d) {
            const uint32_t j = e->deps[d];
            if (e->stream_of[j] != sk) CUDA_TRY(cudaStreamWaitEvent(st, e->done[j], 0));
        }
        int rc = launch_one(e, i, st);
        if (rc != GFB_OK) return rc;
        CUDA_TRY(cudaEventRecord(e->done[i], st));
    }
    for (uint32_t k = 1; k < e->n_streams; ++k) {
        CUDA_TRY(cudaEventRecord(e->joins[k], e->streams[k]));
        CUDA_TRY(cudaStreamWaitEvent(s0, e->joins[k], 0));
    }
    return GFB_OK;
}

int upload_table(gfb_exe* e, void* const* inputs, void* const* outputs, cudaStream_t s) {
    // kernels read caller buffers with 16-byte vector loads, cp.async and TMA
    for (uint32_t i = 0; i < e->n_in; ++i)
        if (reinterpret_cast<uintptr_t>(inputs[i]) & 15)
            return fail(GFB_ERR_INVALID, "input " + std::to_string(i) + ": device pointer not 16-byte aligned");
    for (uint32_t j = 0; j < e->n_out; ++j)
        if (reinterpret_cast<uintptr_t>(outputs[j]) & 15)
            return fail(GFB_ERR_INVALID, "output " + std::to_string(j) + ": device pointer not 16-byte aligned");
    CUDA_TRY(cudaEventSynchronize(e->tab_done));  // previous run consumed the staging copy
    // the previous run may be in flight on another stream: its kernels still
    // read the device table and the arena this run is about to reuse
    if (e->ran) CUDA_TRY(cudaStreamWaitEvent(s, e->run_done, 0));
    e->htab[GFB_SLOT_ARENA] = e->arena;
    e->htab[GFB_SLOT_CONST] = e->consts;
    for (uint32_t i = 0; i < e->n_in; ++i) e->htab[GFB_SLOT_IO + i] = inputs[i];
    for (uint32_t j = 0; j < e->n_out; ++j) e->htab[GFB_SLOT_IO + e->n_in + j] = outputs[j];
    CUDA_TRY(cudaMemcpyAsync(e->dtab, e->htab, sizeof(void*) * e->n_slots, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaEventRecord(e->tab_done, s));
    return GFB_OK;
}

int mark_done(gfb_exe* e, cudaStream_t s) {
    CUDA_TRY(cudaEventRecord(e->run_done, s));
    e->ran = true;
    return GFB_OK;
}

void drop_host_graph(gfb_exe* e) {
    if (e->hexec) cudaGraphExecDestroy(e->hexec);
    if (e->hgraph) cudaGraphDestroy(e->hgraph);
    e->hexec = nullptr;
    e->hgraph = nullptr;
}

void drop_graphs(gfb_exe* e) {
    if (e->graph) cudaGraphExecDestroy(e->graph);
    e->graph = nullptr;
    drop_host_graph(e);
}

// input pieces in order of their first reader; unread pieces are never copied
void order_pieces(gfb_exe* e) {
    const size_t n = e->launches.size(), np = e->pc_in.size();
    std::vector<uint32_t> first(np, UINT32_MAX);
    for (size_t i = n; i-- > 0;)
        for (uint32_t r = e->rd_off[i]; r < e->rd_off[i + 1]; ++r) first[e->rd[r]] = (uint32_t)i;
    e->in_order.clear();
    for (size_t i = 0; i < n; ++i)
        for (uint32_t q = 0; q < np; ++q)
            if (first[q] == i) e->in_order.push_back(q);
}

void release_io(gfb_exe* e) {
    for (void* p : e->dev_in) cudaFree(p);
    for (void* p : e->dev_out) cudaFree(p);
    for (cudaEvent_t ev : e->in_ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : e->wr_ev)
        if (ev) cudaEventDestroy(ev);
    if (e->io_fork) cudaEventDestroy(e->io_fork);
    if (e->h2d_join) cudaEventDestroy(e->h2d_join);
    if (e->d2h_join) cudaEventDestroy(e->d2h_join);
    if (e->h2d) cudaStreamDestroy(e->h2d);
    if (e->d2h) cudaStreamDestroy(e->d2h);
    e->dev_in.clear();
    e->dev_out.clear();
    e->in_ev.clear();
    e->wr_ev.clear();
    e->io_fork = e->h2d_join = e->d2h_join = nullptr;
    e->h2d = e->d2h = nullptr;
    e->io_set = false;
}

// Capture of a host-buffer run: the inputs' H2D copies run on their own
// stream in first-use order, and each launch waits only for the copies of
// the inputs it reads, so the step starts as soon as its first operand has
// arrived and later inputs (weights, targets) cross PCIe under the forward
// pass; each result's D2H copy runs on a third stream right after the last
// launch writing it, under the rest of the step.
int launch_all_io(gfb_exe* e, cudaStream_t s0, const void* const* hin, void* const* hout) {
    // One stream unless GFB_HOST_STREAMS=multi: measured on config E, the
    // host-buffer graph captured over the multi-stream schedule ran 10-25 ms
    // slower than the same launches in order on one stream (the device-only
    // graph runs the same either way).
    const char* hs = getenv("GFB_HOST_STREAMS");
    const bool multi = e->n_streams > 1 && hs && std::string(hs) == "multi";
    CUDA_TRY(cudaEventRecord(e->io_fork, s0));
    CUDA_TRY(cudaStreamWaitEvent(e->h2d, e->io_fork, 0));
    CUDA_TRY(cudaStreamWaitEvent(e->d2h, e->io_fork, 0));
    if (multi)
        for (uint32_t k = 1; k < e->n_streams; ++k) CUDA_TRY(cudaStreamWaitEvent(e->streams[k], e->io_fork, 0));
    const size_t npc = e->pc_in.size();
    for (uint32_t p : e->in_order) {
        const uint32_t i = e->pc_in[p];
        CUDA_TRY(cudaMemcpyAsync((char*)e->dev_in[i] + e->pc_off[p], (const char*)hin[i] + e->pc_off[p], e->pc_len[p],
                                 cudaMemcpyHostToDevice, e->h2d));
        CUDA_TRY(cudaEventRecord(e->in_ev[p], e->h2d));
    }
    std::vector<char> waited(npc * (size_t)(multi ? e->n_streams : 1), 0);
    for (size_t i = 0; i < e->launches.size(); ++i) {
        const uint32_t sk = multi ? e->stream_of[i] : 0;
        cudaStream_t st = sk == 0 ? s0 : e->streams[sk];
        if (multi)
            for (uint32_t d = e->dep_off[i]; d < e->dep_off[i + 1]; ++d) {
                const uint32_t j = e->deps[d];
                if (e->stream_of[j] != sk) CUDA_TRY(cudaStreamWaitEvent(st, e->done[j], 0));
            }
        for (uint32_t r = e->rd_off[i]; r < e->rd_off[i + 1]; ++r) {
            char& w = waited[(size_t)sk * npc + e->rd[r]];
            if (!w) CUDA_TRY(cudaStreamWaitEvent(st, e->in_ev[e->rd[r]], 0));
            w = 1;
        }
        int rc = launch_one(e, i, st);
        if (rc != GFB_OK) return rc;
        if (multi) CUDA_TRY(cudaEventRecord(e->done[i], st));
        if (e->wr_ev[i]) {
            CUDA_TRY(cudaEventRecord(e->wr_ev[i], st));
            CUDA_TRY(cudaStreamWaitEvent(e->d2h, e->wr_ev[i], 0));
            for (uint32_t j = 0; j < e->n_out; ++j)
                if (e->out_writer[j] == i)
                    CUDA_TRY(cudaMemcpyAsync(hout[j], e->dev_out[j], e->out_bytes[j], cudaMemcpyDeviceToHost, e->d2h));
        }
    }
    if (multi)
        for (uint32_t k = 1; k < e->n_streams; ++k) {
            CUDA_TRY(cudaEventRecord(e->joins[k], e->streams[k]));
            CUDA_TRY(cudaStreamWaitEvent(s0, e->joins[k], 0));
        }
    CUDA_TRY(cudaEventRecord(e->h2d_join, e->h2d));
    CUDA_TRY(cudaStreamWaitEvent(s0, e->h2d_join, 0));
    CUDA_TRY(cudaEventRecord(e->d2h_join, e->d2h));
    CUDA_TRY(cudaStreamWaitEvent(s0, e->d2h_join, 0));
    return GFB_OK;
}

// The memcpy nodes of a captured host-buffer graph, found by their device
// staging address, so later runs retarget them at new host buffers.
bool find_copy_nodes(gfb_exe* e) {
    size_t n = 0;
    if (cudaGraphGetNodes(e->hgraph, nullptr, &n) != cudaSuccess) return false;
    std::vector<cudaGraphNode_t> nodes(n);
    if (cudaGraphGetNodes(e->hgraph, nodes.data(), &n) != cudaSuccess) return false;
    e->h2d_node.assign(e->pc_in.size(), nullptr);
    e->d2h_node.assign(e->n_out, nullptr);
    for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nd, &t) != cudaSuccess || t != cudaGraphNodeTypeMemcpy) continue;
        cudaMemcpy3DParms p;
        if (cudaGraphMemcpyNodeGetParams(nd, &p) != cudaSuccess) return false;
        const char* dst = (const char*)p.dstPtr.ptr + p.dstPos.x;
        for (uint32_t q : e->in_order)
            if (dst == (const char*)e->dev_in[e->pc_in[q]] + e->pc_off[q]) e->h2d_node[q] = nd;
        for (uint32_t j = 0; j < e->n_out; ++j)
            if (p.srcPtr.ptr == e->dev_out[j]) e->d2h_node[j] = nd;
    }
    for (uint32_t q : e->in_order)
        if (!e->h2d_node[q]) return false;
    for (uint32_t j = 0; j < e->n_out; ++j)
        if (!e->d2h_node[j]) return false;
    return true;
}

void release_schedule(gfb_exe* e) {
    for (size_t k = 1; k < e->streams.size(); ++k) cudaStreamDestroy(e->streams[k]);
    for (cudaEvent_t ev : e->done) cudaEventDestroy(ev);
    for (size_t k = 1; k < e->joins.size(); ++k) cudaEventDestroy(e->joins[k]);
    if (e->fork) cudaEventDestroy(e->fork);
    e->streams.clear();
    e->done.clear();
    e->joins.clear();
    e->fork = nullptr;
    e->n_streams = 1;
}

void release(gfb_exe* e) {
    if (e->ran && e->run_done) cudaEventSynchronize(e->run_done);
    if (e->nccl_reg && e->comm && g_nccl.CommDeregister) g_nccl.CommDeregister(e->comm->comm, e->nccl_reg);
    release_schedule(e);
    drop_graphs(e);
    release_io(e);
    if (e->run_done) cudaEventDestroy(e->run_done);
    if (e->capture_stream) cudaStreamDestroy(e->capture_stream);
    if (e->tab_done) cudaEventDestroy(e->tab_done);
    if (e->htab) cudaFreeHost(e->htab);
    if (e->dtab) cudaFree(e->dtab);
    if (e->consts) cudaFree(e->consts);
    if (e->arena) cudaFree(e->arena);
    delete e;
}

}  // namespace

extern "C" {

const char* gfb_last_error(void) { return g_err.c_str(); }

int gfb_init(int device) {
    int count = 0;
    CUDA_TRY(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(GFB_ERR_INVALID, "device index out of range");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(GFB_ERR_UNSUPPORTED, std::string("need an sm_100 (B200) device, found ") + prop.name);
    return GFB_OK;
}

int gfb_device_info(int* sm_major, int* sm_minor, int* num_sms) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
    *sm_major = prop.major;
    *sm_minor = prop.minor;
    *num_sms = prop.multiProcessorCount;
    return GFB_OK;
}

int gfb_exe_create(const gfb_plan* plan, gfb_exe** out) {
    if (!plan || !out) return fail(GFB_ERR_INVALID, "null plan");
    gfb_exe* e = new gfb_exe();
    auto bail = [&](int rc) {
        release(e);
        return rc;
    };
    if (cudaGetDevice(&e->device) != cudaSuccess) return bail(fail(GFB_ERR_CUDA, "cudaGetDevice failed"));
    e->n_in = plan->n_inputs;
    e->n_out = plan->n_outputs;
    e->n_slots = GFB_SLOT_IO + e->n_in + e->n_out;
    e->use_graph = (plan->flags & GFB_PLAN_CUDA_GRAPH) != 0;
    e->comm = (gfb_comm*)plan->comm;
    cudaError_t err;
    if (plan->arena_bytes && (err = cudaMalloc(&e->arena, plan->arena_bytes)) != cudaSuccess)
        return bail(fail(GFB_ERR_CUDA, std::string("arena cudaMalloc: ") + cudaGetErrorString(err)));
    if (plan->const_bytes) {
        if ((err = cudaMalloc(&e->consts, plan->const_bytes)) != cudaSuccess)
            return bail(fail(GFB_ERR_CUDA, std::string("constant pool cudaMalloc: ") + cudaGetErrorString(err)));
        if ((err = cudaMemcpy(e->consts, plan->const_data, plan->const_bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
            return bail(fail(GFB_ERR_CUDA, std::string("constant upload: ") + cudaGetErrorString(err)));
    }
    if ((err = cudaMalloc(&e->dtab, sizeof(void*) * e->n_slots)) != cudaSuccess ||
        (err = cudaMallocHost(&e->htab, sizeof(void*) * e->n_slots)) != cudaSuccess ||
        (err = cudaEventCreateWithFlags(&e->tab_done, cudaEventDisableTiming)) != cudaSuccess ||
        (err = cudaEventCreateWithFlags(&e->run_done, cudaEventDisableTiming)) != cudaSuccess ||
        (err = cudaStreamCreateWithFlags(&e->capture_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(fail(GFB_ERR_CUDA, std::string("executable setup: ") + cudaGetErrorString(err)));
    e->launches.assign(plan->launches, plan->launches + plan->n_launches);
    e->args.assign((const unsigned char*)plan->args, (const unsigned char*)plan->args + plan->args_bytes);
    e->fns.resize(e->launches.size(), nullptr);
    for (size_t i = 0; i < e->launches.size(); ++i) {
        const gfb_launch& L = e->launches[i];
        if ((uint64_t)L.arg_offset + L.arg_size > plan->args_bytes || L.arg_size < sizeof(void*))
            return bail(fail(GFB_ERR_INVALID, "launch argument block out of range"));
        // Every argument block starts with the device pointer table.
        std::memcpy(e->args.data() + L.arg_offset, &e->dtab, sizeof(void*));
        if (L.kind == GFB_K_ALLREDUCE) {
            if (!e->comm) return bail(fail(GFB_ERR_INVALID, "all-reduce launch without a communicator"));
            continue;
        }
        if (L.kind == GFB_K_MEMSET) continue;
        e->fns[i] = kernel_for(L.kind);
        if (!e->fns[i]) return bail(fail(GFB_ERR_INVALID, "unknown kernel kind " + std::to_string(L.kind)));
        if (L.kind == GFB_K_DOT_TC32 || L.kind == GFB_K_DOT_TC32W || L.kind == GFB_K_DOT_TC32P) {
            // Tensor maps need fixed addresses: the split planes live in the arena.
            gfb_tc_args* a = (gfb_tc_args*)(e->args.data() + L.arg_offset);
            const uint64_t refs[4] = {a->a_hi, a->a_lo, a->b_hi, a->b_lo};
            for (int t = 0; t < 4; ++t) {
                if ((refs[t] >> 56) != GFB_SLOT_ARENA)
                    return bail(fail(GFB_ERR_INVALID, "tensor-core operand planes must live in the arena"));
                void* addr = (char*)e->arena + (refs[t] & ((1ull << 56) - 1));
                const int64_t rows = t < 2 ? a->M : a->N, kp = t < 2 ? a->kp_a : a->kp_b;
                const int64_t ld_mn = t < 2 ? a->a_ld_mn : a->b_ld_mn;
                const uint32_t box_rows = (t >= 2 && L.kind == GFB_K_DOT_TC32W) ? 256 : 128;
                if (ld_mn > 0) {
                    if (L.kind != GFB_K_DOT_TC32P)
                        return bail(fail(GFB_ERR_INVALID, "MN-major operands need the CTA-pair GEMM"));
                    if (!encode_mn_map(addr, rows, a->K, ld_mn, a->tmap[t]))
                        return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled (MN-major operand) failed"));
                } else if (!encode_plane_map(addr, rows, kp, box_rows, a->tmap[t]))
                    return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled failed"));
            }
        }
        if (L.kind == GFB_K_DOT_F16P) {
            gfb_tc_args* a = (gfb_tc_args*)(e->args.data() + L.arg_offset);
            const uint64_t refs[4] = {a->a_hi, a->a_lo, a->b_hi, a->b_lo};
            for (int t = 0; t < 4; ++t) {
                if ((refs[t] >> 56) != GFB_SLOT_ARENA)
                    return bail(fail(GFB_ERR_INVALID, "tensor-core operand planes must live in the arena"));
                void* addr = (char*)e->arena + (refs[t] & ((1ull << 56) - 1));
                const int64_t rows = t < 2 ? a->M : a->N, kp = t < 2 ? a->kp_a : a->kp_b;
                const int64_t ld_mn = t < 2 ? a->a_ld_mn : a->b_ld_mn;
                const bool ok = ld_mn > 0 ? encode_mn16_map(addr, rows, a->K, ld_mn, a->tmap[t]) : encode_plane16_map(addr, rows, kp, a->tmap[t]);
                if (!ok) return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled (fp16 plane) failed"));
            }
        }
        if (L.kind == GFB_K_CONV_TCXH64 || L.kind == GFB_K_CONV_TCXH128) {
            gfb_tcxh_args* a = (gfb_tcxh_args*)(e->args.data() + L.arg_offset);
            const uint64_t refs[4] = {a->a_hi, a->a_lo, a->b_hi, a->b_lo};
            void* addr[4];
            for (int t = 0; t < 4; ++t) {
                if ((refs[t] >> 56) != GFB_SLOT_ARENA)
                    return bail(fail(GFB_ERR_INVALID, "TMA convolution operands must live in the arena"));
                addr[t] = (char*)e->arena + (refs[t] & ((1ull << 56) - 1));
            }
            for (int t = 0; t < 2; ++t)
                if (!encode_act16_map(addr[t], a->a_dims, a->a_strides, (uint32_t)(a->BX * a->sx), (uint32_t)(a->BY * a->sy),
                                      (uint32_t)a->BNI, (uint32_t)a->sx, (uint32_t)a->sy, a->tmap[t]))
                    return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled (fp16 activation box) failed"));
            for (int t = 2; t < 4; ++t)
                if (!encode_plane16_map(addr[t], a->N, a->K, a->tmap[t], L.kind == GFB_K_CONV_TCXH64 ? 64 : 128))
                    return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled (fp16 filter plane) failed"));
        }
        if (L.kind == GFB_K_CONV_TCGWH64 || L.kind == GFB_K_CONV_TCGWH128) {
            gfb_tcgwh_args* a = (gfb_tcgwh_args*)(e->args.data() + L.arg_offset);
            const uint64_t refs[4] = {a->a_hi, a->a_lo, a->b_hi, a->b_lo};
            for (int t = 0; t < 4; ++t) {
                if ((refs[t] >> 56) != GFB_SLOT_ARENA)
                    return bail(fail(GFB_ERR_INVALID, "TMA convolution operands must live in the arena"));
                void* addr = (char*)e->arena + (refs[t] & ((1ull << 56) - 1));
                if (!encode_act16_map(addr, t < 2 ? a->a_dims : a->b_dims, t < 2 ? a->a_strides : a->b_strides, (uint32_t)a->BX,
                                      (uint32_t)a->BY, (uint32_t)a->BNI, 1, 1, a->tmap[t]))
                    return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled (fp16 gradient box) failed"));
            }
        }
        if (L.kind == GFB_K_CONV_TCX64 || L.kind == GFB_K_CONV_TCX128) {
            gfb_tcx_args* a = (gfb_tcx_args*)(e->args.data() + L.arg_offset);
            const uint64_t refs[3] = {a->a, a->b_hi, a->b_lo};
            void* addr[3];
            for (int t = 0; t < 3; ++t) {
                if ((refs[t] >> 56) != GFB_SLOT_ARENA)
                    return bail(fail(GFB_ERR_INVALID, "TMA convolution operands must live in the arena"));
                addr[t] = (char*)e->arena + (refs[t] & ((1ull << 56) - 1));
            }
            if (!encode_act_map(addr[0], a->a_dims, a->a_strides, (uint32_t)(a->BX * a->sx), (uint32_t)(a->BY * a->sy),
                                (uint32_t)a->BNI, (uint32_t)a->sx, (uint32_t)a->sy, a->tmap[0]))
                return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled (activation box) failed"));
            for (int t = 1; t < 3; ++t)
                if (!encode_plane_map(addr[t], a->N, a->K, L.kind == GFB_K_CONV_TCX64 ? 64 : 128, a->tmap[t]))
                    return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled failed"));
        }
        if (L.kind == GFB_K_CONV_TCGG64 || L.kind == GFB_K_CONV_TCGG128) {
            gfb_tcgg_args* a = (gfb_tcgg_args*)(e->args.data() + L.arg_offset);
            const uint64_t refs[2] = {a->b_hi, a->b_lo};
            for (int t = 0; t < 2; ++t) {
                if ((refs[t] >> 56) != GFB_SLOT_ARENA)
                    return bail(fail(GFB_ERR_INVALID, "tensor-core operand planes must live in the arena"));
                void* addr = (char*)e->arena + (refs[t] & ((1ull << 56) - 1));
                if (!encode_plane_map(addr, a->N, a->kp_b, L.kind == GFB_K_CONV_TCGG64 ? 64 : 128, a->tmap[t]))
                    return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled failed"));
            }
        }
        if (L.kind == GFB_K_CONV_TCG64 || L.kind == GFB_K_CONV_TCG128 || L.kind == GFB_K_CONV_STEM64) {
            gfb_tcg_args* a = (gfb_tcg_args*)(e->args.data() + L.arg_offset);
            const uint64_t refs[2] = {a->b_hi, a->b_lo};
            for (int t = 0; t < 2; ++t) {
                if ((refs[t] >> 56) != GFB_SLOT_ARENA)
                    return bail(fail(GFB_ERR_INVALID, "tensor-core operand planes must live in the arena"));
                void* addr = (char*)e->arena + (refs[t] & ((1ull << 56) - 1));
                const int64_t kp = L.kind == GFB_K_CONV_STEM64 ? a->pad[1] : a->K;  // stem: plane pitch in pad[1]
                if (!encode_plane_map(addr, a->N, kp, L.kind == GFB_K_CONV_TCG128 ? 128 : 64, a->tmap[t]))
                    return bail(fail(GFB_ERR_CUDA, "cuTensorMapEncodeTiled failed"));
            }
        }
    }
    // Opt every kernel in to the largest dynamic shared memory any of its
    // launches needs (the attribute is per function, not per launch).
    for (size_t i = 0; i < e->launches.size(); ++i) {
        if (!e->fns[i] || e->launches[i].smem < 40 * 1024) continue;  // leave room for static smem
        uint32_t need = 0;
        for (size_t j = 0; j < e->launches.size(); ++j)
            if (e->fns[j] == e->fns[i]) need = need > e->launches[j].smem ? need : e->launches[j].smem;
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, e->fns[i]) == cudaSuccess && (uint32_t)fa.maxDynamicSharedSizeBytes >= need) continue;
        err = cudaFuncSetAttribute(e->fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
        if (err != cudaSuccess) return bail(fail(GFB_ERR_CUDA, std::string("smem attribute: ") + cudaGetErrorString(err)));
    }
    // Optional NCCL user-buffer registration of the arena (every all-reduce
    // bucket lives there), so collectives can skip the internal staging copy.
    if (e->comm && e->arena && g_nccl.CommRegister) {
        const char* reg = getenv("GFB_NCCL_REGISTER");
        if (reg && reg[0] == '1') {
            ncclResult_t r = g_nccl.CommRegister(e->comm->comm, e->arena, plan->arena_bytes, &e->nccl_reg);
            if (r != 0) return bail(nccl_fail(r, "ncclCommRegister"));
        }
    }
    *out = e;
    return GFB_OK;
}

namespace {
// NVTX range for the host side of a run (graph upload / capture / launch);
// free unless a tool (nsys, ncu --nvtx) is attached
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

int gfb_exe_run(gfb_exe* e, void* const* inputs, void* const* outputs, void* stream) {
    if (!e) return fail(GFB_ERR_INVALID, "null executable");
    NvtxRange range("gfb_exe_run");
    std::lock_guard<std::mutex> lk(e->mu);
    cudaStream_t s = stream ? (cudaStream_t)stream : cudaStreamPerThread;
    int rc = upload_table(e, inputs, outputs, s);
    if (rc != GFB_OK) return rc;
    if (!e->use_graph) {
        rc = launch_all(e, s);
        return rc != GFB_OK ? rc : mark_done(e, s);
    }
    if (!e->graph) {
        // Capture on a private stream: nothing executes during capture, and
        // the instantiated graph is then launched on the caller's stream.
        CUDA_TRY(cudaStreamBeginCapture(e->capture_stream, cudaStreamCaptureModeThreadLocal));
        rc = e->n_streams > 1 ? launch_all_streams(e, e->capture_stream) : launch_all(e, e->capture_stream);
        cudaGraph_t g = nullptr;
        cudaError_t end = cudaStreamEndCapture(e->capture_stream, &g);
        if (rc != GFB_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (end != cudaSuccess) return fail(GFB_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(end));
        cudaError_t inst = cudaGraphInstantiate(&e->graph, g, 0);
        cudaGraphDestroy(g);
        if (inst != cudaSuccess) return fail(GFB_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(inst));
    }
    CUDA_TRY(cudaGraphLaunch(e->graph, s));
    return mark_done(e, s);
}

int gfb_exe_run_one(gfb_exe* e, uint32_t index, void* const* inputs, void* const* outputs, void* stream) {
    if (!e || index >= e->launches.size()) return fail(GFB_ERR_INVALID, "bad launch index");
    std::lock_guard<std::mutex> lk(e->mu);
    cudaStream_t s = stream ? (cudaStream_t)stream : cudaStreamPerThread;
    int rc = upload_table(e, inputs, outputs, s);
    if (rc != GFB_OK) return rc;
    rc = launch_one(e, index, s);
    return rc != GFB_OK ? rc : mark_done(e, s);
}

int gfb_exe_set_io(gfb_exe* e, const uint64_t* in_bytes, const uint64_t* out_bytes, const uint32_t* read_offsets,
                   const uint32_t* reads, const uint32_t* out_writer) {
    if (!e || (e->n_in && !in_bytes) || (e->n_out && (!out_bytes || !out_writer)) || !read_offsets)
        return fail(GFB_ERR_INVALID, "gfb_exe_set_io: null argument");
    std::lock_guard<std::mutex> lk(e->mu);
    const size_t n = e->launches.size();
    if (read_offsets[0] != 0) return fail(GFB_ERR_INVALID, "gfb_exe_set_io: read_offsets[0] must be 0");
    for (size_t i = 0; i < n; ++i) {
        if (read_offsets[i + 1] < read_offsets[i]) return fail(GFB_ERR_INVALID, "gfb_exe_set_io: offsets not monotone");
        for (uint32_t r = read_offsets[i]; r < read_offsets[i + 1]; ++r)
            if (reads[r] >= e->n_in) return fail(GFB_ERR_INVALID, "gfb_exe_set_io: input index out of range");
    }
    for (uint32_t j = 0; j < e->n_out; ++j)
        if (out_writer[j] >= n) return fail(GFB_ERR_INVALID, "gfb_exe_set_io: every result needs a writing launch");
    if (e->ran) CUDA_TRY(cudaEventSynchronize(e->run_done));  // a host-buffer run may still use the old buffers
    drop_graphs(e);
    release_io(e);
    e->in_bytes.assign(in_bytes, in_bytes + e->n_in);
    e->out_bytes.assign(out_bytes, out_bytes + e->n_out);
    e->rd_off.assign(read_offsets, read_offsets + n + 1);
    e->rd.assign(reads, reads + read_offsets[n]);
    e->out_writer.assign(out_writer, out_writer + e->n_out);
    e->pc_in.resize(e->n_in);
    e->pc_off.assign(e->n_in, 0);
    e->pc_len.assign(e->in_bytes.begin(), e->in_bytes.end());
    for (uint32_t k = 0; k < e->n_in; ++k) e->pc_in[k] = k;  // one piece per input
    order_pieces(e);
    e->dev_in.assign(e->n_in, nullptr);
    e->dev_out.assign(e->n_out, nullptr);
    e->in_ev.assign(e->n_in, nullptr);
    e->wr_ev.assign(n, nullptr);
    auto bail = [&](cudaError_t err) {
        release_io(e);
        return fail(GFB_ERR_CUDA, std::string("gfb_exe_set_io: ") + cudaGetErrorString(err));
    };
    cudaError_t err;
    for (uint32_t i = 0; i < e->n_in; ++i)
        if ((err = cudaMalloc(&e->dev_in[i], e->in_bytes[i] ? e->in_bytes[i] : 1)) != cudaSuccess ||
            (err = cudaEventCreateWithFlags(&e->in_ev[i], cudaEventDisableTiming)) != cudaSuccess)
            return bail(err);
    for (uint32_t j = 0; j < e->n_out; ++j) {
        if ((err = cudaMalloc(&e->dev_out[j], e->out_bytes[j] ? e->out_bytes[j] : 1)) != cudaSuccess) return bail(err);
        if (!e->wr_ev[e->out_writer[j]] &&
            (err = cudaEventCreateWithFlags(&e->wr_ev[e->out_writer[j]], cudaEventDisableTiming)) != cudaSuccess)
            return bail(err);
    }
    if ((err = cudaEventCreateWithFlags(&e->io_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (err = cudaEventCreateWithFlags(&e->h2d_join, cudaEventDisableTiming)) != cudaSuccess ||
        (err = cudaEventCreateWithFlags(&e->d2h_join, cudaEventDisableTiming)) != cudaSuccess ||
        (err = cudaStreamCreateWithFlags(&e->h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (err = cudaStreamCreateWithFlags(&e->d2h, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(err);
    e->io_set = true;
    return GFB_OK;
}

int gfb_exe_set_io_pieces(gfb_exe* e, uint32_t n_pieces, const uint32_t* piece_input, const uint64_t* piece_offset,
                          const uint64_t* piece_bytes, const uint32_t* read_offsets, const uint32_t* reads) {
    if (!e || !read_offsets || (n_pieces && (!piece_input || !piece_offset || !piece_bytes)))
        return fail(GFB_ERR_INVALID, "gfb_exe_set_io_pieces: null argument");
    std::lock_guard<std::mutex> lk(e->mu);
    if (!e->io_set) return fail(GFB_ERR_INVALID, "gfb_exe_set_io_pieces before gfb_exe_set_io");
    const size_t n = e->launches.size();
    for (uint32_t p = 0; p < n_pieces; ++p)
        if (piece_input[p] >= e->n_in || piece_offset[p] + piece_bytes[p] > e->in_bytes[piece_input[p]])
            return fail(GFB_ERR_INVALID, "gfb_exe_set_io_pieces: piece outside its input");
    if (read_offsets[0] != 0) return fail(GFB_ERR_INVALID, "gfb_exe_set_io_pieces: read_offsets[0] must be 0");
    for (size_t i = 0; i < n; ++i) {
        if (read_offsets[i + 1] < read_offsets[i]) return fail(GFB_ERR_INVALID, "gfb_exe_set_io_pieces: offsets not monotone");
        for (uint32_t r = read_offsets[i]; r < read_offsets[i + 1]; ++r)
            if (reads[r] >= n_pieces) return fail(GFB_ERR_INVALID, "gfb_exe_set_io_pieces: piece index out of range");
    }
    if (e->ran) CUDA_TRY(cudaEventSynchronize(e->run_done));
    drop_host_graph(e);
    for (cudaEvent_t ev : e->in_ev) cudaEventDestroy(ev);
    e->in_ev.assign(n_pieces, nullptr);
    for (uint32_t p = 0; p < n_pieces; ++p) CUDA_TRY(cudaEventCreateWithFlags(&e->in_ev[p], cudaEventDisableTiming));
    e->pc_in.assign(piece_input, piece_input + n_pieces);
    e->pc_off.assign(piece_offset, piece_offset + n_pieces);
    e->pc_len.assign(piece_bytes, piece_bytes + n_pieces);
    e->rd_off.assign(read_offsets, read_offsets + n + 1);
    e->rd.assign(reads, reads + read_offsets[n]);
    order_pieces(e);
    return GFB_OK;
}

int gfb_exe_run_host(gfb_exe* e, const void* const* host_inputs, void* const* host_outputs, void* stream) {
    if (!e) return fail(GFB_ERR_INVALID, "null executable");
    NvtxRange range("gfb_exe_run_host");
    std::lock_guard<std::mutex> lk(e->mu);
    if (!e->io_set) return fail(GFB_ERR_INVALID, "gfb_exe_run_host before gfb_exe_set_io");
    bool known = e->hexec != nullptr;  // the buffers of the previous run were checked then
    for (uint32_t i = 0; known && i < e->n_in; ++i) known = e->cur_hin[i] == host_inputs[i];
    for (uint32_t j = 0; known && j < e->n_out; ++j) known = e->cur_hout[j] == host_outputs[j];
    for (uint32_t i = 0; !known && i < e->n_in + e->n_out; ++i) {
        const void* p = i < e->n_in ? host_inputs[i] : host_outputs[i - e->n_in];
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeHost) {
            cudaGetLastError();
            return fail(GFB_ERR_INVALID, "gfb_exe_run_host: host buffer " + std::to_string(i) + " is not page-locked");
        }
    }
    cudaStream_t s = stream ? (cudaStream_t)stream : cudaStreamPerThread;
    int rc = upload_table(e, e->dev_in.data(), e->dev_out.data(), s);
    if (rc != GFB_OK) return rc;
    if (!e->use_graph) {  // in order on one stream
        for (uint32_t i = 0; i < e->n_in; ++i)
            CUDA_TRY(cudaMemcpyAsync(e->dev_in[i], host_inputs[i], e->in_bytes[i], cudaMemcpyHostToDevice, s));
        rc = launch_all(e, s);
        if (rc != GFB_OK) return rc;
        for (uint32_t j = 0; j < e->n_out; ++j)
            CUDA_TRY(cudaMemcpyAsync(host_outputs[j], e->dev_out[j], e->out_bytes[j], cudaMemcpyDeviceToHost, s));
        return mark_done(e, s);
    }
    bool same = e->hexec != nullptr;
    for (uint32_t i = 0; same && i < e->n_in; ++i) same = e->cur_hin[i] == host_inputs[i];
    for (uint32_t j = 0; same && j < e->n_out; ++j) same = e->cur_hout[j] == host_outputs[j];
    if (e->hexec && !same) {
        // retarget the copy nodes at this call's host buffers (once the
        // previous launch of the graph has finished with the old ones)
        CUDA_TRY(cudaEventSynchronize(e->run_done));
        for (uint32_t q : e->in_order) {
            const uint32_t i = e->pc_in[q];
            if (e->cur_hin[i] != host_inputs[i])
                CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(e->hexec, e->h2d_node[q], (char*)e->dev_in[i] + e->pc_off[q],
                                                            (const char*)host_inputs[i] + e->pc_off[q], e->pc_len[q],
                                                            cudaMemcpyHostToDevice));
        }
        for (uint32_t j = 0; j < e->n_out; ++j)
            if (e->cur_hout[j] != host_outputs[j])
                CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(e->hexec, e->d2h_node[j], host_outputs[j], e->dev_out[j],
                                                            e->out_bytes[j], cudaMemcpyDeviceToHost));
    }
    if (!e->hexec) {
        CUDA_TRY(cudaStreamBeginCapture(e->capture_stream, cudaStreamCaptureModeThreadLocal));
        rc = launch_all_io(e, e->capture_stream, host_inputs, host_outputs);
        cudaGraph_t g = nullptr;
        cudaError_t end = cudaStreamEndCapture(e->capture_stream, &g);
        if (rc != GFB_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (end != cudaSuccess) return fail(GFB_ERR_CUDA, std::string("host-run graph capture: ") + cudaGetErrorString(end));
        e->hgraph = g;
        if (!find_copy_nodes(e)) {
            drop_host_graph(e);
            return fail(GFB_ERR_CUDA, "host-run graph: copy nodes not found");
        }
        cudaError_t inst = cudaGraphInstantiate(&e->hexec, g, 0);
        if (inst != cudaSuccess) {
            e->hexec = nullptr;
            drop_host_graph(e);
            return fail(GFB_ERR_CUDA, std::string("host-run graph instantiate: ") + cudaGetErrorString(inst));
        }
    }
    e->cur_hin.assign(host_inputs, host_inputs + e->n_in);
    e->cur_hout.assign(host_outputs, host_outputs + e->n_out);
    CUDA_TRY(cudaGraphLaunch(e->hexec, s));
    return mark_done(e, s);
}

int gfb_exe_num_launches(const gfb_exe* e) { return e ? (int)e->launches.size() : 0; }

int gfb_kernel_load(const void* cubin, const char* name, const void** kernel) {
    if (!cubin || !name || !kernel) return fail(GFB_ERR_INVALID, "null argument");
    cudaLibrary_t lib = nullptr;
    CUDA_TRY(cudaLibraryLoadData(&lib, cubin, nullptr, nullptr, 0, nullptr, nullptr, 0));
    cudaKernel_t k = nullptr;
    CUDA_TRY(cudaLibraryGetKernel(&k, lib, name));
    *kernel = (const void*)k;  // the library stays loaded for the life of the process
    return GFB_OK;
}

int gfb_exe_set_schedule(gfb_exe* e, uint32_t n_streams, const uint32_t* stream_of, const uint32_t* dep_offsets,
                         const uint32_t* deps) {
    if (!e || n_streams == 0 || n_streams > 16 || (n_streams > 1 && (!stream_of || !dep_offsets)))
        return fail(GFB_ERR_INVALID, "bad schedule");
    std::lock_guard<std::mutex> lk(e->mu);
    const size_t n = e->launches.size();
    release_schedule(e);
    drop_graphs(e);
    if (n_streams == 1) return GFB_OK;
    for (size_t i = 0; i < n; ++i) {
        if (stream_of[i] >= n_streams) return fail(GFB_ERR_INVALID, "schedule: stream index out of range");
        for (uint32_t d = dep_offsets[i]; d < dep_offsets[i + 1]; ++d)
            if (deps[d] >= i) return fail(GFB_ERR_INVALID, "schedule: a launch may only wait for earlier launches");
    }
    e->stream_of.assign(stream_of, stream_of + n);
    e->dep_off.assign(dep_offsets, dep_offsets + n + 1);
    e->deps.assign(deps, deps + dep_offsets[n]);
    e->streams.assign(n_streams, nullptr);
    e->streams[0] = e->capture_stream;
    e->joins.assign(n_streams, nullptr);
    e->done.assign(n, nullptr);
    e->n_streams = n_streams;
    for (uint32_t k = 1; k < n_streams; ++k) {
        CUDA_TRY(cudaStreamCreateWithFlags(&e->streams[k], cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&e->joins[k], cudaEventDisableTiming));
    }
    for (size_t i = 0; i < n; ++i) CUDA_TRY(cudaEventCreateWithFlags(&e->done[i], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming));
    return GFB_OK;
}

int gfb_exe_set_kernel(gfb_exe* e, uint32_t index, const void* kernel, uint32_t smem) {
    if (!e || index >= e->launches.size()) return fail(GFB_ERR_INVALID, "bad launch index");
    std::lock_guard<std::mutex> lk(e->mu);
    const uint32_t kind = e->launches[index].kind;
    if (!((kind >= GFB_K_EW_F32 && kind <= GFB_K_EW1_F64) || kind == GFB_K_ROWJIT))
        return fail(GFB_ERR_INVALID, "only fused elementwise / row launches take a runtime-compiled kernel");
    if (kernel && smem >= 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    e->fns[index] = kernel;
    e->launches[index].smem = smem;
    drop_graphs(e);
    return GFB_OK;
}

int gfb_exe_destroy(gfb_exe* e) {
    if (!e) return GFB_OK;
    release(e);  // waits for the last run, whatever stream it was launched on
    return GFB_OK;
}

int gfb_comm_unique_id(void* unique_id_128) {
    int rc = load_nccl();
    if (rc != GFB_OK) return rc;
    ncclResult_t r = g_nccl.GetUniqueId(unique_id_128);
    return r ? nccl_fail(r, "ncclGetUniqueId") : GFB_OK;
}

int gfb_comm_create(int nranks, int rank, const void* unique_id_128, gfb_comm** out) {
    int rc = load_nccl();
    if (rc != GFB_OK) return rc;
    gfb_comm* c = new gfb_comm();
    c->nranks = nranks;
    c->rank = rank;
    NcclUniqueId id;
    std::memcpy(id.internal, unique_id_128, 128);
    InitRankFn init = (InitRankFn)g_nccl.CommInitRank;
    ncclResult_t r = init(&c->comm, nranks, id, rank);
    if (r) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    *out = c;
    return GFB_OK;
}

int gfb_comm_destroy(gfb_comm* c) {
    if (!c) return GFB_OK;
    if (c->comm) g_nccl.CommDestroy(c->comm);
    delete c;
    return GFB_OK;
}

}  // extern "C"
