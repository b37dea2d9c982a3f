// capi.cu -- extern "C" boundary of libps_b200.so (declared in include/ps_b200.h).
//
// Validates arguments (PS_ERR_INVALID, mapped to ValueError by the Python
// layer), launches the sm_100a kernels on the caller's stream, and converts
// CUDA failures into PS_ERR_CUDA with a message.  Nothing here allocates
// device memory: buffers and workspaces are owned by the caller.

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "../../include/ps_b200.h"
#include "common.cuh"
#include "group.h"
#include "ps_internal.h"
#include "sampler.h"

namespace {

thread_local char g_err[512] = "";
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_status(cudaError_t e, const char* what, int launches) {
    if (e != cudaSuccess) return fail(PS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    g_launches += launches;
    return PS_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int64_t kMaxN = (int64_t)1 << 30;

#define CHECK_ARG(cond, ...) \
    do {                     \
        if (!(cond)) return fail(PS_ERR_INVALID, __VA_ARGS__); \
    } while (0)

// ---- small drop-in kernels -------------------------------------------------

__global__ void __launch_bounds__(1024) chunk_update_kernel(const float4* __restrict__ xyz, double px, double py,
                                                            double pz, double* md, int64_t lo, int64_t hi,
                                                            double* best_out, int64_t* arg_out) {
    __shared__ uint64_t wk[32];
    __shared__ uint32_t wi[32];
    uint64_t bkey = 0;
    uint32_t bidx = 0xffffffffu;
    for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
        const float4 v = xyz[j];
        const double d = ps::sqdist(px, py, pz, (double)v.x, (double)v.y, (double)v.z);
        double m = md[j];
        if (d < m) { m = d; md[j] = d; }
        const uint64_t key = (uint64_t)__double_as_longlong(m);
        if (bidx == 0xffffffffu || key > bkey) { bkey = key; bidx = (uint32_t)(j - lo); }
    }
    ps::ArgMax a = ps::warp_argmax(bkey, bidx);
    if ((threadIdx.x & 31) == 0) { wk[threadIdx.x >> 5] = a.key; wi[threadIdx.x >> 5] = a.idx; }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int nw = blockDim.x >> 5;
        const uint64_t k = threadIdx.x < nw ? wk[threadIdx.x] : 0;
        const uint32_t i = threadIdx.x < nw ? wi[threadIdx.x] : 0xffffffffu;
        a = ps::warp_argmax(k, i);
        if (threadIdx.x == 0) {
            if (a.idx == 0xffffffffu) { *best_out = -1.0; *arg_out = -1; }
            else { *best_out = __longlong_as_double((long long)a.key); *arg_out = lo + a.idx; }
        }
    }
}

// out4[b][t] = xyz4[b][idx[b][t]] (w = 0): the next set-abstraction stage's
// input, in sample order
__global__ void gather_xyz4_kernel(const float4* __restrict__ xyz, const int64_t* __restrict__ idx, int64_t idx_ld,
                                   int64_t B, int64_t N, int64_t n, float4* __restrict__ out) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < B * n; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = g / n, t = g - b * n;
        const int64_t j = idx[b * idx_ld + t];
        float4 v = (j >= 0 && j < N) ? xyz[b * N + j] : make_float4(0.f, 0.f, 0.f, 0.f);
        v.w = 0.f;
        out[g] = v;
    }
}

__global__ void __launch_bounds__(1024) first_untaken_kernel(const uint8_t* taken, int64_t N, int64_t* out) {
    __shared__ unsigned long long best;
    if (threadIdx.x == 0) best = ~0ull;
    __syncthreads();
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        if (!taken[j]) { atomicMin(&best, (unsigned long long)j); break; }
    }
    __syncthreads();
    if (threadIdx.x == 0) *out = best == ~0ull ? -1 : (int64_t)best;
}

}  // namespace

extern "C" {

int ps_version(void) { return 1; }
const char* ps_last_error(void) { return g_err; }
int64_t ps_launch_count(void) { return g_launches.load(); }

int ps_fps_loop(const float* xyz4, int64_t B, int64_t N, double* md, uint8_t* taken, int64_t* out_idx,
                double* curve, int64_t ld_out, int64_t k_start, const int64_t* k_start_dev, int64_t n_total,
                void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN, "invalid batch shape B=%lld N=%lld", (long long)B, (long long)N);
    CHECK_ARG(n_total <= ld_out, "n_total %lld exceeds row stride %lld", (long long)n_total, (long long)ld_out);
    CHECK_ARG(k_start_dev || k_start >= 1, "k_start must be >= 1");
    CHECK_ARG(xyz4 && md && taken && out_idx && curve, "null pointer");
    ps::FpsArgs a = {};
    a.xyz = reinterpret_cast<const float4*>(xyz4);
    a.md = md; a.taken = taken; a.out_idx = out_idx; a.curve = curve;
    a.k_start_dev = k_start_dev; a.seed_dev = nullptr;
    a.N = N; a.ld_out = ld_out; a.k_start = k_start; a.k_stop = n_total; a.seed = 0; a.fresh = 0;
    return cuda_status(ps::launch_fps(a, B, S(stream)), "fps_loop", 1);
}

int64_t ps_set_fps_inflight(int64_t clouds) { return ps::fps_set_inflight(clouds); }

int ps_fps(const float* xyz4, int64_t B, int64_t N, double* md, uint8_t* taken, int64_t* out_idx, double* curve,
           int64_t ld_out, int64_t k_stop, int64_t seed, const int64_t* seed_dev, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN, "invalid batch shape B=%lld N=%lld", (long long)B, (long long)N);
    CHECK_ARG(k_stop >= 1 && k_stop <= ld_out && k_stop <= N, "k_stop %lld out of range", (long long)k_stop);
    CHECK_ARG(seed_dev || (seed >= 0 && seed < N), "seed index %lld out of range", (long long)seed);
    CHECK_ARG(xyz4 && md && taken && out_idx && curve, "null pointer");
    ps::FpsArgs a = {};
    a.xyz = reinterpret_cast<const float4*>(xyz4);
    a.md = md; a.taken = taken; a.out_idx = out_idx; a.curve = curve;
    a.k_start_dev = nullptr; a.seed_dev = seed_dev;
    a.N = N; a.ld_out = ld_out; a.k_start = 1; a.k_stop = k_stop; a.seed = seed; a.fresh = 1;
    return cuda_status(ps::launch_fps(a, B, S(stream)), "fps", 1);
}

// ---- K1 point-split: one cloud split over G ranks ----------------------------------

int64_t ps_fps_mailbox_bytes(int64_t B, int32_t G) {
    if (B < 1 || G < 1) return 0;
    return B * 3 * (int64_t)G * ps::kMbRecs * ps::kRecU4 * (int64_t)sizeof(uint4);
}

int ps_fps_split_plan(int64_t N, int64_t B, int32_t G, int32_t Gl, int32_t* C_out, int32_t* P_out) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN && G >= 1 && G <= ps::kMaxRanks && Gl >= 1 && Gl <= G,
              "invalid split shape (1 <= Gl <= G <= %d)", ps::kMaxRanks);
    int C = 0, P = 0;
    if (!ps::fps_res_plan(N, B * Gl, G, &C, &P))
        return fail(PS_ERR_UNSUPPORTED, "no co-resident cluster plan for N=%lld over %d ranks (%d per launch)",
                    (long long)N, G, Gl);
    if (C_out) *C_out = C;
    if (P_out) *P_out = P;
    return PS_OK;
}

int ps_fps_split(const float* xyz4, int64_t B, int64_t N, double* md, uint8_t* taken, int64_t* out_idx, double* curve,
                 int64_t ld_out, int64_t k_stop, int64_t seed, int32_t G, int32_t g_base, int32_t Gl,
                 void* const* mbox_dev, uint32_t seq_base, int32_t all_write, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN, "invalid batch shape B=%lld N=%lld", (long long)B, (long long)N);
    CHECK_ARG(k_stop >= 1 && k_stop <= ld_out && k_stop <= N, "k_stop %lld out of range", (long long)k_stop);
    CHECK_ARG(seed >= 0 && seed < N, "seed index %lld out of range", (long long)seed);
    CHECK_ARG(G >= 1 && G <= ps::kMaxRanks && Gl >= 1 && g_base >= 0 && g_base + Gl <= G,
              "invalid ranks G=%d g_base=%d Gl=%d (G <= %d: one warp lane per rank)", G, g_base, Gl, ps::kMaxRanks);
    CHECK_ARG(G == 1 || mbox_dev != nullptr, "mailbox pointer array required for G > 1");
    CHECK_ARG((uint64_t)seq_base + (uint64_t)k_stop < 0xffffffffull, "sequence space exhausted; reset the mailboxes");
    CHECK_ARG(xyz4 && md && taken && out_idx && curve, "null pointer");
    int C = 0, P = 0;
    if (!ps::fps_res_plan(N, B * Gl, G, &C, &P))
        return fail(PS_ERR_UNSUPPORTED, "no co-resident cluster plan for N=%lld over %d ranks (%d per launch)",
                    (long long)N, G, Gl);
    ps::FpsArgs a = {};
    a.xyz = reinterpret_cast<const float4*>(xyz4);
    a.md = md; a.taken = taken; a.out_idx = out_idx; a.curve = curve;
    a.N = N; a.ld_out = ld_out; a.k_start = 1; a.k_stop = k_stop; a.seed = seed; a.fresh = 1;
    ps::FpsRanks rk = {};
    rk.G = G; rk.Gl = Gl; rk.g_base = g_base; rk.all_write = all_write; rk.seq_base = seq_base;
    rk.mbox = reinterpret_cast<uint4* const*>(mbox_dev);
    rk.timeout_ns = ps::split_timeout_ns();
    return cuda_status(ps::launch_fps_res(a, rk, B, C, P, S(stream)), "fps_split", 1);
}

int ps_fps_split_loop(const float* xyz4, int64_t B, int64_t N, double* md, uint8_t* taken, int64_t* out_idx,
                      double* curve, int64_t ld_out, int64_t k_start, const int64_t* k_start_dev, int64_t n_total,
                      int32_t G, int32_t g_base, int32_t Gl, void* const* mbox_dev, uint32_t seq_base,
                      int32_t all_write, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN, "invalid batch shape B=%lld N=%lld", (long long)B, (long long)N);
    CHECK_ARG(n_total >= 1 && n_total <= ld_out && n_total <= N, "n_total %lld out of range", (long long)n_total);
    CHECK_ARG(k_start_dev || k_start >= 1, "k_start must be >= 1");
    CHECK_ARG(G >= 1 && G <= ps::kMaxRanks && Gl >= 1 && g_base >= 0 && g_base + Gl <= G,
              "invalid ranks G=%d g_base=%d Gl=%d (G <= %d: one warp lane per rank)", G, g_base, Gl, ps::kMaxRanks);
    CHECK_ARG(G == 1 || mbox_dev != nullptr, "mailbox pointer array required for G > 1");
    CHECK_ARG((uint64_t)seq_base + (uint64_t)n_total < 0xffffffffull, "sequence space exhausted; reset the mailboxes");
    CHECK_ARG(xyz4 && md && taken && out_idx && curve, "null pointer");
    int C = 0, P = 0;
    if (!ps::fps_res_plan(N, B * Gl, G, &C, &P))
        return fail(PS_ERR_UNSUPPORTED, "no co-resident cluster plan for N=%lld over %d ranks (%d per launch)",
                    (long long)N, G, Gl);
    ps::FpsArgs a = {};
    a.xyz = reinterpret_cast<const float4*>(xyz4);
    a.md = md; a.taken = taken; a.out_idx = out_idx; a.curve = curve;
    a.k_start_dev = k_start_dev;
    a.N = N; a.ld_out = ld_out; a.k_start = k_start; a.k_stop = n_total; a.seed = 0; a.fresh = 0;
    ps::FpsRanks rk = {};
    rk.G = G; rk.Gl = Gl; rk.g_base = g_base; rk.all_write = all_write; rk.seq_base = seq_base;
    rk.mbox = reinterpret_cast<uint4* const*>(mbox_dev);
    rk.timeout_ns = ps::split_timeout_ns();
    return cuda_status(ps::launch_fps_res(a, rk, B, C, P, S(stream)), "fps_split_loop", 1);
}

int ps_device_alloc(int64_t bytes, int32_t fill_byte, void** dev_ptr_out) {
    CHECK_ARG(bytes > 0 && dev_ptr_out, "invalid allocation request");
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)bytes);
    if (e != cudaSuccess) return fail(PS_ERR_CUDA, "cudaMalloc(%lld): %s", (long long)bytes, cudaGetErrorString(e));
    if (fill_byte >= 0) {
        e = cudaMemset(p, fill_byte & 0xff, (size_t)bytes);
        if (e != cudaSuccess) {
            cudaFree(p);
            return fail(PS_ERR_CUDA, "cudaMemset: %s", cudaGetErrorString(e));
        }
    }
    *dev_ptr_out = p;
    return PS_OK;
}

int ps_device_free(void* dev_ptr) {
    const cudaError_t e = cudaFree(dev_ptr);
    if (e != cudaSuccess) return fail(PS_ERR_CUDA, "cudaFree: %s", cudaGetErrorString(e));
    return PS_OK;
}

int ps_ipc_handle(const void* dev_ptr, void* handle_out) {
    CHECK_ARG(dev_ptr && handle_out, "null pointer");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
    if (e != cudaSuccess) return fail(PS_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    memcpy(handle_out, &h, sizeof(h));
    return PS_OK;
}

int ps_ipc_open(const void* handle, void** dev_ptr_out) {
    CHECK_ARG(handle && dev_ptr_out, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(PS_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return PS_OK;
}

int ps_ipc_close(void* dev_ptr) {
    const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return fail(PS_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return PS_OK;
}

int ps_fps_update_chunk(const float* xyz4, int64_t N, double px, double py, double pz, double* md, int64_t lo,
                        int64_t hi, double* best_out, int64_t* arg_out, void* stream) {
    CHECK_ARG(N >= 1 && lo >= 0 && lo <= hi && hi <= N, "invalid slice [%lld, %lld)", (long long)lo, (long long)hi);
    chunk_update_kernel<<<1, 1024, 0, S(stream)>>>(reinterpret_cast<const float4*>(xyz4), px, py, pz, md, lo, hi,
                                                  best_out, arg_out);
    return cuda_status(cudaGetLastError(), "fps_update_chunk", 1);
}

int ps_gather_xyz4(const float* xyz4, const int64_t* idx, int64_t idx_ld, int64_t B, int64_t N, int64_t n,
                   float* out4, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && n >= 0 && n <= idx_ld, "invalid gather shape");
    CHECK_ARG(xyz4 && idx && out4, "null pointer");
    if (n == 0) return PS_OK;
    const unsigned g = (unsigned)std::min<int64_t>(148 * 8, (B * n + 255) / 256);
    gather_xyz4_kernel<<<g, 256, 0, S(stream)>>>(reinterpret_cast<const float4*>(xyz4), idx, idx_ld, B, N, n,
                                                 reinterpret_cast<float4*>(out4));
    return cuda_status(cudaGetLastError(), "gather_xyz4", 1);
}

int ps_first_untaken(const uint8_t* taken, int64_t N, int64_t* out, void* stream) {
    CHECK_ARG(N >= 0, "invalid N");
    first_untaken_kernel<<<1, 1024, 0, S(stream)>>>(taken, N, out);
    return cuda_status(cudaGetLastError(), "first_untaken", 1);
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static int grid_max_cells(int64_t N) {
    const int64_t c = 4 * N + 64;
    return (int)(c < ((int64_t)1 << 24) ? c : ((int64_t)1 << 24));
}

int64_t ps_excl_workspace_bytes(int64_t B, int64_t N, int64_t cap_edges, int32_t method) {
    size_t s = 0;
    if (method == 0) {
        s += align_up(sizeof(uint32_t) * B * cap_edges) * 2;
        s += align_up(sizeof(double) * B * cap_edges);
        s += align_up(sizeof(unsigned long long) * B);
    } else {
        const int64_t mc = grid_max_cells(N);
        s += align_up(sizeof(ps::GridParams) * B);
        s += align_up(sizeof(int) * B * (mc + 1));
        s += align_up(sizeof(int) * B * mc);
        s += align_up(sizeof(int32_t) * B * N) * 2;
        s += align_up(sizeof(float4) * B * N);
        s += align_up(sizeof(unsigned long long) * B) * 2;  // evals, spill
    }
    s += align_up(sizeof(int32_t) * B * N) * 2;
    s += align_up(sizeof(unsigned));
    return (int64_t)s;
}

int64_t ps_excl_row_stride(int64_t N, int64_t cap_entries) {
    return N >= 1 ? ps::ell_row_stride(cap_entries, N) : 0;
}

int64_t ps_excl_grid_evals_offset(int64_t B, int64_t N) {
    const int64_t mc = grid_max_cells(N);
    size_t s = 0;
    s += align_up(sizeof(ps::GridParams) * B);
    s += align_up(sizeof(int) * B * (mc + 1));
    s += align_up(sizeof(int) * B * mc);
    s += align_up(sizeof(int32_t) * B * N) * 2;
    s += align_up(sizeof(float4) * B * N);
    return (int64_t)s;
}

int ps_excl_build(const float* xyz4, int64_t B, int64_t N, const double* r2_levels, int32_t L, int64_t levels_ld,
                  int64_t* indptr, int32_t* nbr, double* d2, int32_t* counts, int64_t cap_entries, void* work,
                  int64_t cap_edges, int32_t* status, int32_t method, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN, "invalid batch shape");
    CHECK_ARG(L >= 1 && L <= levels_ld && L <= 32, "invalid level count %d (1..32)", L);
    CHECK_ARG(cap_entries >= N && cap_entries < ((int64_t)1 << 31), "cap_entries must be in [N, 2^31)");
    CHECK_ARG(cap_edges >= 1, "cap_edges must be >= 1");
    CHECK_ARG(method >= 0 && method <= 2, "method must be 0 (brute force), 1 (grid) or 2 (grid, strided bucket rows)");
    CHECK_ARG(method != 2 || ps::ell_row_stride(cap_entries, N) <= 65535, "row stride too large");
    CHECK_ARG(work && status && indptr && nbr && d2 && counts, "null pointer");
    unsigned char* w = static_cast<unsigned char*>(work);
    ps::ExclWork ew = {};
    ps::GridWork gw = {};
    ew.cap_edges = cap_edges;
    if (method == 0) {
        ew.edge_i = reinterpret_cast<uint32_t*>(w); w += align_up(sizeof(uint32_t) * B * cap_edges);
        ew.edge_j = reinterpret_cast<uint32_t*>(w); w += align_up(sizeof(uint32_t) * B * cap_edges);
        ew.edge_d2 = reinterpret_cast<double*>(w); w += align_up(sizeof(double) * B * cap_edges);
        ew.edge_count = reinterpret_cast<unsigned long long*>(w); w += align_up(sizeof(unsigned long long) * B);
    } else {
        const int64_t mc = grid_max_cells(N);
        gw.max_cells = (int)mc;
        gw.params = reinterpret_cast<ps::GridParams*>(w); w += align_up(sizeof(ps::GridParams) * B);
        gw.cell_start = reinterpret_cast<int*>(w); w += align_up(sizeof(int) * B * (mc + 1));
        gw.cursor = reinterpret_cast<int*>(w); w += align_up(sizeof(int) * B * mc);
        gw.cell_of = reinterpret_cast<int32_t*>(w); w += align_up(sizeof(int32_t) * B * N);
        gw.sorted_idx = reinterpret_cast<int32_t*>(w); w += align_up(sizeof(int32_t) * B * N);
        gw.sorted_xyz = reinterpret_cast<float4*>(w); w += align_up(sizeof(float4) * B * N);
        gw.evals = reinterpret_cast<unsigned long long*>(w); w += align_up(sizeof(unsigned long long) * B);
        ew.spill = reinterpret_cast<unsigned long long*>(w); w += align_up(sizeof(unsigned long long) * B);
    }
    ew.deg = reinterpret_cast<int32_t*>(w); w += align_up(sizeof(int32_t) * B * N);
    ew.long_rows = reinterpret_cast<int32_t*>(w); w += align_up(sizeof(int32_t) * B * N);
    ew.long_count = reinterpret_cast<unsigned*>(w);
    ew.status = status;
    ps::CsrView csr = {indptr, nbr, d2, counts, cap_entries, N, L};
    return cuda_status(ps::launch_excl_build(reinterpret_cast<const float4*>(xyz4), B, N, r2_levels, L, levels_ld,
                                             csr, ew, gw, method, S(stream)),
                       "excl_build", ps::excl_build_launches(N, method));
}

int64_t ps_csr_fill_workspace_bytes(int64_t M, int64_t N) {
    if (M < 0 || N < 1) return 0;
    return (int64_t)ps::csr_fill_ws_bytes(M, N);
}

int ps_csr_fill(const int32_t* ei, const int32_t* ej, const double* ed, int64_t M, const int64_t* indptr, int64_t N,
                int64_t* out_idx, double* out_d2, void* work, int64_t work_bytes, void* stream) {
    CHECK_ARG(N >= 1 && N < ((int64_t)1 << 31) && M >= 0 && 2 * M < ((int64_t)1 << 31), "invalid sizes");
    CHECK_ARG(indptr && out_idx && out_d2 && (M == 0 || (ei && ej && ed)), "null pointer");
    CHECK_ARG(work && work_bytes >= ps_csr_fill_workspace_bytes(M, N), "workspace too small (ps_csr_fill_workspace_bytes)");
    return cuda_status(ps::launch_csr_fill(ei, ej, ed, M, indptr, N, out_idx, out_d2, work, (size_t)work_bytes,
                                           S(stream)),
                       "csr_fill", M > 0 ? 3 : 1);
}

int ps_csr_sort_rows(int64_t* indptr, int32_t* nbr, double* d2, int64_t cap_entries, int64_t B, int64_t N,
                     void* work, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN, "invalid batch shape");
    CHECK_ARG(work != nullptr, "null workspace");
    unsigned char* w = static_cast<unsigned char*>(work);
    ps::ExclWork ew = {};
    ew.long_rows = reinterpret_cast<int32_t*>(w);
    w += align_up(sizeof(int32_t) * B * N);
    ew.long_count = reinterpret_cast<unsigned*>(w);
    ps::CsrView csr = {indptr, nbr, d2, nullptr, cap_entries, N, 0};
    return cuda_status(ps::launch_sort_rows(csr, B, ew, S(stream)), "csr_sort_rows", 2);
}

int ps_level_counts(const int64_t* indptr, const double* d2, int64_t cap_entries, int64_t B, int64_t N,
                    const double* r2_levels, int32_t L, int64_t levels_ld, int32_t* counts, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && L >= 1, "invalid shape");
    ps::CsrView csr = {const_cast<int64_t*>(indptr), nullptr, const_cast<double*>(d2), counts, cap_entries, N, L};
    return cuda_status(ps::launch_level_counts(csr, B, r2_levels, levels_ld, S(stream)), "level_counts", 1);
}

int ps_thresholds(const double* prefix_curve, int64_t curve_ld, int64_t B, int64_t k0, int64_t n, int32_t nseg,
                  const int64_t* d_host, int32_t mode, const double* pow_tab, const double* given_curve,
                  int64_t given_ld, const double* extra_r2_host, int32_t n_extra, double* R_out, double* r2_levels,
                  int64_t levels_ld, void* stream) {
    CHECK_ARG(nseg >= 1 && nseg <= ps::kMaxSeg, "nseg must be in [1, %d]", ps::kMaxSeg);
    CHECK_ARG(n_extra >= 0 && n_extra <= ps::kMaxExtra, "at most %d extra radii", ps::kMaxExtra);
    CHECK_ARG(k0 >= 2 && k0 <= n, "prefix length k0=%lld must be in [2, n]", (long long)k0);
    CHECK_ARG(levels_ld >= nseg + n_extra, "levels_ld too small");
    CHECK_ARG(mode == 0 ? pow_tab != nullptr : given_curve != nullptr, "missing estimator input");
    ps::ThreshArgs a = {};
    a.prefix_curve = prefix_curve; a.curve_ld = curve_ld; a.pow_tab = pow_tab;
    a.given_curve = given_curve; a.given_ld = given_ld; a.mode = mode;
    a.k0 = k0; a.n = n; a.nseg = nseg;
    for (int s = 0; s < nseg; ++s) {
        CHECK_ARG(d_host[s] >= 0 && d_host[s] < n, "d[%d] out of range", s);
        a.d[s] = d_host[s];
    }
    a.n_extra = n_extra;
    for (int e = 0; e < n_extra; ++e) a.extra_r2[e] = extra_r2_host[e];
    a.R_out = R_out; a.r2_levels = r2_levels; a.levels_ld = levels_ld;
    return cuda_status(ps::launch_thresholds(a, B, S(stream)), "thresholds", 1);
}

int ps_thresholds_mlp(const double* prefix_curve, int64_t curve_ld, int64_t B, int64_t k0, int64_t n, int32_t nseg,
                      const int64_t* d_host, const double* mlp_weights, const double* extra_r2_host, int32_t n_extra,
                      double* R_out, double* r2_levels, int64_t levels_ld, void* stream) {
    CHECK_ARG(nseg >= 1 && nseg <= ps::kMaxSeg, "nseg must be in [1, %d]", ps::kMaxSeg);
    CHECK_ARG(n_extra >= 0 && n_extra <= ps::kMaxExtra, "at most %d extra radii", ps::kMaxExtra);
    CHECK_ARG(k0 >= 3 && k0 <= n, "the MLP estimator needs k0 in [3, n] (k0=%lld)", (long long)k0);
    CHECK_ARG(levels_ld >= nseg + n_extra, "levels_ld too small");
    CHECK_ARG(mlp_weights != nullptr, "missing MLP weights");
    ps::ThreshArgs a = {};
    a.prefix_curve = prefix_curve; a.curve_ld = curve_ld; a.mode = 2; a.mlp = mlp_weights;
    a.k0 = k0; a.n = n; a.nseg = nseg;
    for (int s = 0; s < nseg; ++s) {
        CHECK_ARG(d_host[s] >= 0 && d_host[s] < n, "d[%d] out of range", s);
        a.d[s] = d_host[s];
    }
    a.n_extra = n_extra;
    for (int e = 0; e < n_extra; ++e) a.extra_r2[e] = extra_r2_host[e];
    a.R_out = R_out; a.r2_levels = r2_levels; a.levels_ld = levels_ld;
    return cuda_status(ps::launch_thresholds(a, B, S(stream)), "thresholds_mlp", 1);
}

int64_t ps_sampler_workspace_bytes(int64_t B, int64_t N, int32_t nseg) {
    (void)nseg;
    return (int64_t)ps::sampler_global_ws_bytes(B, N, true);
}

int ps_sample_predicted(const int64_t* indptr, const int32_t* nbr, int64_t cap_entries, const int32_t* counts,
                        int32_t L, const int32_t* seg_level_rows_host, const int64_t* boundaries_host, int32_t nseg,
                        int64_t* out_idx, int64_t ld_out, int64_t k0, int64_t n_total, int64_t B, int64_t N,
                        uint64_t* state_io, int32_t pick_lowest, int64_t* reached, int32_t* exhausted,
                        int32_t* entered, void* work, const int32_t* excl_status, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN, "invalid batch shape");
    CHECK_ARG(nseg >= 1 && nseg <= ps::kMaxSeg, "nseg must be in [1, %d]", ps::kMaxSeg);
    CHECK_ARG(k0 >= 0 && k0 <= n_total && n_total <= ld_out && n_total <= N, "invalid k0/n_total");
    CHECK_ARG(boundaries_host[nseg - 1] == n_total,
              "last segment boundary must equal n_total (got %lld, n_total %lld)",
              (long long)boundaries_host[nseg - 1], (long long)n_total);
    ps::SampArgs a = {};
    a.indptr = indptr; a.nbr = nbr; a.cap_entries = cap_entries; a.counts = counts; a.L = L; a.nseg = nseg;
    for (int s = 0; s < nseg; ++s) {
        CHECK_ARG(seg_level_rows_host[s] >= 0 && seg_level_rows_host[s] < L, "seg_level_rows[%d] out of range", s);
        CHECK_ARG(s == 0 || boundaries_host[s] >= boundaries_host[s - 1], "boundaries must be non-decreasing");
        a.seg_level_rows[s] = seg_level_rows_host[s];
        a.boundaries[s] = boundaries_host[s];
    }
    a.k0 = k0; a.n_total = n_total; a.N = N; a.out_idx = out_idx; a.ld_out = ld_out; a.state_io = state_io;
    a.pick_lowest = pick_lowest; a.reached = reached; a.exhausted = exhausted; a.entered = entered;
    a.excl_status = excl_status;
    CHECK_ARG(work != nullptr, "sampler workspace required (ps_sampler_workspace_bytes)");
    a.gws = static_cast<unsigned char*>(work);
    a.B = B;
    return cuda_status(ps::launch_sampler(a, B, S(stream)), "sample_predicted", 1);
}

int ps_earlyterm_scan(const int64_t* indptr, const int32_t* nbr, const double* d2, int64_t cap_entries,
                      const int32_t* lvl1_counts, int64_t counts_stride, const uint8_t* taken, double* md, int64_t B,
                      int64_t N, int64_t lo, int64_t hi, void* stream) {
    CHECK_ARG(B >= 1 && 0 <= lo && lo <= hi && hi <= N, "invalid range");
    if (lo == hi) return PS_OK;
    ps::EtScanArgs a = {};
    a.indptr = indptr; a.nbr = nbr; a.d2 = d2; a.cap_entries = cap_entries; a.lvl1_counts = lvl1_counts;
    a.counts_stride = counts_stride; a.taken = taken; a.md = md; a.reached = nullptr; a.n_total = 0;
    a.B = B; a.N = N; a.lo = lo; a.hi = hi;
    return cuda_status(ps::launch_et_scan(a, S(stream)), "earlyterm_scan", 1);
}

int ps_early_termination_prepare(const int64_t* indptr, const int32_t* nbr, const double* d2, int64_t cap_entries,
                                 const int32_t* lvl1_counts, int64_t counts_stride, uint8_t* taken, double* md,
                                 const int64_t* out_idx, int64_t ld_out, const int64_t* reached, int64_t n_total,
                                 int64_t B, int64_t N, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1, "invalid shape");
    ps::EtArgs a = {};
    a.indptr = indptr; a.nbr = nbr; a.d2 = d2; a.cap_entries = cap_entries; a.lvl1_counts = lvl1_counts;
    a.counts_stride = counts_stride; a.taken = taken; a.md = md; a.out_idx = out_idx; a.ld_out = ld_out;
    a.reached = reached; a.n_total = n_total; a.B = B; a.N = N;
    return cuda_status(ps::launch_et(a, S(stream)), "early_termination_prepare", ps::et_launches());
}

int ps_early_termination_shard(const int64_t* indptr, const int32_t* nbr, const double* d2, int64_t cap_entries,
                               const int32_t* lvl1_counts, int64_t counts_stride, uint8_t* taken, double* md,
                               const int64_t* out_idx, int64_t ld_out, const int64_t* reached, int64_t n_total,
                               int64_t B, int64_t N, int64_t lo, int64_t hi, void* stream) {
    CHECK_ARG(B >= 1 && N >= 1, "invalid shape");
    CHECK_ARG(0 <= lo && lo < hi && hi <= N, "invalid point range [%lld, %lld)", (long long)lo, (long long)hi);
    CHECK_ARG(indptr && nbr && d2 && lvl1_counts && taken && md && out_idx && reached, "null pointer");
    ps::EtArgs a = {};
    a.indptr = indptr; a.nbr = nbr; a.d2 = d2; a.cap_entries = cap_entries; a.lvl1_counts = lvl1_counts;
    a.counts_stride = counts_stride; a.taken = taken; a.md = md; a.out_idx = out_idx; a.ld_out = ld_out;
    a.reached = reached; a.n_total = n_total; a.B = B; a.N = N;
    return cuda_status(ps::launch_et_shard(a, lo, hi, S(stream)), "early_termination_shard", 3);
}

int ps_excl_build_shard(const float* xyz4, int64_t B, int64_t N, const double* r2_levels, int32_t L, int64_t levels_ld,
                        int64_t row_lo, int64_t row_hi, int64_t spill_lo, int64_t spill_hi, int64_t* indptr,
                        int32_t* nbr, double* d2, int32_t* counts, int64_t cap_entries, void* work, int32_t* status,
                        void* stream) {
    CHECK_ARG(B >= 1 && N >= 1 && N <= kMaxN, "invalid batch shape");
    CHECK_ARG(L >= 1 && L <= levels_ld && L <= 32, "invalid level count %d (1..32)", L);
    CHECK_ARG(cap_entries >= N && cap_entries < ((int64_t)1 << 31), "cap_entries must be in [N, 2^31)");
    const int64_t stride = ps::ell_row_stride(cap_entries, N);
    CHECK_ARG(stride <= 65535, "row stride too large");
    CHECK_ARG(0 <= row_lo && row_lo < row_hi && row_hi <= N, "invalid row range [%lld, %lld)", (long long)row_lo,
              (long long)row_hi);
    CHECK_ARG(0 <= spill_lo && spill_lo < spill_hi && spill_hi <= cap_entries - N * stride,
              "spill range must lie in [0, %lld)", (long long)(cap_entries - N * stride));
    CHECK_ARG(work && status && indptr && nbr && d2 && counts, "null pointer");
    unsigned char* w = static_cast<unsigned char*>(work);
    ps::ExclWork ew = {};
    ps::GridWork gw = {};
    ew.cap_edges = 1;
    const int64_t mc = grid_max_cells(N);
    gw.max_cells = (int)mc;
    gw.params = reinterpret_cast<ps::GridParams*>(w); w += align_up(sizeof(ps::GridParams) * B);
    gw.cell_start = reinterpret_cast<int*>(w); w += align_up(sizeof(int) * B * (mc + 1));
    gw.cursor = reinterpret_cast<int*>(w); w += align_up(sizeof(int) * B * mc);
    gw.cell_of = reinterpret_cast<int32_t*>(w); w += align_up(sizeof(int32_t) * B * N);
    gw.sorted_idx = reinterpret_cast<int32_t*>(w); w += align_up(sizeof(int32_t) * B * N);
    gw.sorted_xyz = reinterpret_cast<float4*>(w); w += align_up(sizeof(float4) * B * N);
    gw.evals = reinterpret_cast<unsigned long long*>(w); w += align_up(sizeof(unsigned long long) * B);
    ew.spill = reinterpret_cast<unsigned long long*>(w); w += align_up(sizeof(unsigned long long) * B);
    ew.deg = reinterpret_cast<int32_t*>(w); w += align_up(sizeof(int32_t) * B * N);
    ew.long_rows = reinterpret_cast<int32_t*>(w); w += align_up(sizeof(int32_t) * B * N);
    ew.long_count = reinterpret_cast<unsigned*>(w);
    ew.status = status;
    ps::CsrView csr = {indptr, nbr, d2, counts, cap_entries, N, L, row_lo, row_hi, spill_lo, spill_hi};
    return cuda_status(ps::launch_excl_build(reinterpret_cast<const float4*>(xyz4), B, N, r2_levels, L, levels_ld,
                                             csr, ew, gw, 2, S(stream)),
                       "excl_build_shard", ps::excl_build_launches(N, 2));
}

int ps_ball_query_rf(const int64_t* indptr, const int32_t* nbr, const double* d2, int64_t cap_entries,
                     const int32_t* counts, int32_t L, int32_t level, const int64_t* centroids, int64_t cent_ld,
                     int64_t B, int64_t N, int64_t n, int32_t k, int32_t* idx_out, double* dist_out, int32_t* cnt_out,
                     const int32_t* excl_status, void* stream) {
    CHECK_ARG(k >= 1 && k <= 128, "k must be in [1, 128]");
    CHECK_ARG(level >= 0 && level < L, "level %d out of range [0, %d)", level, L);
    ps::BqArgs a = {};
    a.indptr = indptr; a.nbr = nbr; a.d2 = d2; a.cap_entries = cap_entries; a.counts = counts; a.L = L;
    a.level = level; a.centroids = centroids; a.cent_ld = cent_ld; a.B = B; a.N = N; a.n = n; a.k = k;
    a.idx_out = idx_out; a.dist_out = dist_out; a.cnt_out = cnt_out; a.status = excl_status;
    if (B * n == 0) return PS_OK;
    return cuda_status(ps::launch_bq_rf(a, S(stream)), "ball_query_rf", 1);
}

int ps_ball_query_naive(const float* xyz4, const int64_t* centroids, int64_t cent_ld, int64_t B, int64_t N, int64_t n,
                        double r2, int32_t k, int32_t* idx_out, double* dist_out, int32_t* cnt_out, void* stream) {
    CHECK_ARG(k >= 1 && k <= 128, "k must be in [1, 128]");
    CHECK_ARG(r2 > 0.0, "radius must be positive");
    ps::BqArgs a = {};
    a.xyz = reinterpret_cast<const float4*>(xyz4);
    a.centroids = centroids; a.cent_ld = cent_ld; a.B = B; a.N = N; a.n = n; a.k = k; a.r2 = r2;
    a.idx_out = idx_out; a.dist_out = dist_out; a.cnt_out = cnt_out;
    if (B * n == 0) return PS_OK;
    return cuda_status(ps::launch_bq_naive(a, S(stream)), "ball_query_naive", 1);
}

int ps_knn_naive(const float* xyz4, const int64_t* queries, int64_t q_ld, int64_t nq, const int64_t* pool,
                 int64_t pool_ld, int64_t npool, int64_t B, int64_t N, int32_t k, int32_t* idx_out, double* dist_out,
                 int32_t* cnt_out, void* stream) {
    CHECK_ARG(k >= 1 && k <= 16, "k must be in [1, 16]");
    CHECK_ARG(npool >= 1, "empty pool");
    ps::KnnArgs a = {};
    a.xyz = reinterpret_cast<const float4*>(xyz4);
    a.queries = queries; a.q_ld = q_ld; a.nq = nq; a.pool = pool; a.pool_ld = pool_ld; a.npool = npool;
    a.B = B; a.N = N; a.k = k; a.idx_out = idx_out; a.dist_out = dist_out; a.cnt_out = cnt_out;
    if (B * nq == 0) return PS_OK;
    return cuda_status(ps::launch_knn_naive(a, S(stream)), "knn_naive", 1);
}

int ps_knn_rf(const float* xyz4, const int64_t* indptr, const int32_t* nbr, const double* d2, int64_t cap_entries,
              const int32_t* lvl1_counts, int64_t counts_stride, const uint8_t* sampled, const int64_t* queries,
              int64_t q_ld, int64_t nq, const int64_t* pool, int64_t pool_ld, int64_t npool, int64_t B, int64_t N,
              int32_t k, int32_t* idx_out, double* dist_out, int32_t* cnt_out, int32_t* fallback_count,
              const int32_t* excl_status, void* stream) {
    CHECK_ARG(k >= 1 && k <= 16, "k must be in [1, 16]");
    CHECK_ARG(npool >= 1, "empty pool");
    ps::KnnArgs a = {};
    a.xyz = reinterpret_cast<const float4*>(xyz4);
    a.queries = queries; a.q_ld = q_ld; a.nq = nq; a.pool = pool; a.pool_ld = pool_ld; a.npool = npool;
    a.sampled = sampled; a.indptr = indptr; a.nbr = nbr; a.d2 = d2; a.cap_entries = cap_entries;
    a.lvl1_counts = lvl1_counts; a.counts_stride = counts_stride; a.B = B; a.N = N; a.k = k;
    a.idx_out = idx_out; a.dist_out = dist_out; a.cnt_out = cnt_out; a.fallback_count = fallback_count;
    a.status = excl_status;
    if (B * nq == 0) return PS_OK;
    return cuda_status(ps::launch_knn_rf(a, S(stream)), "knn_rf", 1);
}

int ps_min_spacing(const float* xyz4, const int64_t* samples, int64_t ld, int64_t n, int64_t B, int64_t N,
                   double* out_d2, void* stream) {
    CHECK_ARG(n >= 1 && B >= 1, "invalid shape");
    ps::SpacingArgs a = {reinterpret_cast<const float4*>(xyz4), samples, ld, n, B, N, out_d2};
    return cuda_status(ps::launch_min_spacing(a, S(stream)), "min_spacing", 1);
}

}  // extern "C"
