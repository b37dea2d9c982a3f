// sampler_v3.cu -- K3c: the predicted-distance bitmap sampler
// (_kernels.py:241-353, sample_predicted) as a per-segment grid of kernels.
//
// The reference keeps one bitmap per segment and clears every accepted
// point's row prefix in the bitmaps of the current and all later segments.
// By the symmetry of the exclusion rows, bit j of segment s at the moment
// segment s is entered is simply "no already-sampled point in j's level-s
// row prefix" -- so instead of maintaining bitmaps, every segment visit
// recomputes availability from the sampled set, grid-wide:
//
//   samp_init    out[k0:] = -1, taken bitmap = FPS prefix, state per cloud
//   per segment s = 0 .. nseg-1 (a cloud takes part when its current segment
//   is s; segments are visited in increasing order, at most once):
//     samp_avail  warp per 32 points: avail(j) = no taken point in row_s(j)
//     samp_adj    thread per available point: its available level-s
//                 neighbours (<= 16, else marked for a full row scan) -- the
//                 only edges the selection can hit
//     samp_visit  one CTA per cloud: the segment pool (available points in
//                 index order), then chunks of 1024 draws:
//                   positions z_t mod (L - t), z_t = splitmix64(state + (t+1)G);
//                   the swap-remove chain as a parallel Fisher-Yates
//                   (sort by position, last-writer links, pointer jumping);
//                   greedy maximal independent set in draw order over the
//                   compressed adjacency (IN if every earlier neighbour is
//                   OUT, OUT if one is IN; accepted points of earlier chunks
//                   are marked in the rank table);
//                   truncation at the segment boundary (draws consumed = last
//                   used accept + 1) or pool exhaustion;
//                 then the accepted points join the taken set and the
//                 segment / entered / exhausted / RNG bookkeeping of
//                 _kernels.py:303-351 runs.
//   samp_final  reached, exhausted, entered, RNG state out.
//
// Bit-exact with the reference: identical candidate order, identical
// acceptance, identical RNG consumption.

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ps_internal.h"
#include "sampler.h"

namespace ps {

namespace {

constexpr uint64_t kGolden3 = 0x9E3779B97F4A7C15ull;
constexpr int kVThreads = 1024;
constexpr int kChunk = 1024;
constexpr int kAdj = 16;
constexpr uint8_t kAdjOverflow = 0xff;
constexpr uint8_t kUnd = 0, kIn = 1, kOut = 2;
constexpr uint16_t kNoRank = 0xffffu;
constexpr uint16_t kAccMark = 0xfffeu;
constexpr int kMaxPred = 8;
constexpr uint8_t kPredOverflow = 0xff;

struct __align__(16) SampState {
    int64_t i;          // samples so far
    uint64_t rng;       // splitmix64 state
    int seg, entered, exhausted, done;
    int64_t pad[5];
};

struct SampWork {
    SampState* st;      // [B]
    uint32_t* taken;    // [B][W]
    uint32_t* avail;    // [B][W]
    int32_t* adj;       // [B][N][kAdj]
    uint8_t* adjcnt;    // [B][N]
    int32_t* gpool;     // [B][N]   (large N)
    uint16_t* grank;    // [B][N]   (large N)
    int64_t W;
};

PS_DEV uint64_t mix64v(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

PS_DEV bool bit(const uint32_t* bm, int32_t j) { return (bm[j >> 5] >> (j & 31)) & 1u; }

PS_DEV int block_scan(int v, int* warp_tot, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int s = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += y;
        }
        warp_tot[lane] = s;
    }
    __syncthreads();
    const int ex = (warp ? warp_tot[warp - 1] : 0) + x - v;
    *total = warp_tot[31];
    __syncthreads();
    return ex;
}

// ---- init / final ------------------------------------------------------------

__global__ void samp_init_kernel(SampArgs a, SampWork w) {
    const int64_t b = blockIdx.x;
    uint32_t* tk = w.taken + b * w.W;
    int64_t* out = a.out_idx + b * a.ld_out;
    for (int64_t x = threadIdx.x; x < w.W; x += blockDim.x) tk[x] = 0u;
    for (int64_t t = a.k0 + threadIdx.x; t < a.n_total; t += blockDim.x) out[t] = -1;
    __syncthreads();
    for (int64_t t = threadIdx.x; t < a.k0; t += blockDim.x) {
        const int32_t p = (int32_t)out[t];
        atomicOr(&tk[p >> 5], 1u << (p & 31));
    }
    if (threadIdx.x == 0) {
        SampState s = {};
        s.i = a.k0;
        s.rng = a.state_io[b];
        int seg = 0;
        while (seg < a.nseg && a.k0 >= a.boundaries[seg]) ++seg;
        s.seg = seg;
        if (seg >= a.nseg) {
            s.done = 1;
            s.exhausted = 1;
            s.entered = 0;
        } else {
            s.entered = 1;
        }
        w.st[b] = s;
    }
}

__global__ void samp_final_kernel(SampArgs a, SampWork w) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= a.B) return;
    const SampState s = w.st[b];
    a.reached[b] = s.i;
    a.exhausted[b] = s.exhausted;
    a.entered[b] = s.entered;
    a.state_io[b] = s.rng;
}

// ---- availability + compressed adjacency for segment s ---------------------------

__global__ void samp_avail_kernel(SampArgs a, SampWork w, int s) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lvl = a.seg_level_rows[s];
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < a.B * w.W; g += nwarps) {
        const int64_t b = g / w.W, word = g - b * w.W;
        const SampState st = w.st[b];
        if (st.done || st.seg != s) continue;
        const uint32_t* tk = w.taken + b * w.W;
        const int64_t j = word * 32 + lane;
        bool av = false;
        if (j < a.N && !bit(tk, (int32_t)j)) {
            av = true;
            const int32_t c = a.counts[(b * a.L + lvl) * a.N + j];
            const int32_t* row = a.nbr + b * a.cap_entries + a.indptr[b * (a.N + 1) + j];
            for (int32_t u = 0; u < c; ++u) {
                if (bit(tk, __ldg(row + u))) { av = false; break; }
            }
        }
        const uint32_t m = __ballot_sync(kFull, av);
        if (lane == 0) w.avail[b * w.W + word] = m;
    }
}

__global__ void samp_adj_kernel(SampArgs a, SampWork w, int s) {
    const int lvl = a.seg_level_rows[s];
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < a.B * a.N;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = g / a.N, j = g - b * a.N;
        const SampState st = w.st[b];
        if (st.done || st.seg != s) continue;
        const uint32_t* av = w.avail + b * w.W;
        if (!bit(av, (int32_t)j)) continue;
        const int32_t c = a.counts[(b * a.L + lvl) * a.N + j];
        const int32_t* row = a.nbr + b * a.cap_entries + a.indptr[b * (a.N + 1) + j];
        int32_t* out = w.adj + g * kAdj;
        int n = 0;
        for (int32_t u = 0; u < c; ++u) {
            const int32_t q = __ldg(row + u);
            if (q != (int32_t)j && bit(av, q)) {
                if (n < kAdj) out[n] = q;
                ++n;
            }
        }
        w.adjcnt[g] = n > kAdj ? kAdjOverflow : (uint8_t)n;
    }
}

// ---- one segment visit per cloud --------------------------------------------------

struct VisitSmem {
    unsigned long long keys[kChunk];  // (position << 32) | draw, sorted
    uint32_t pos[kChunk];
    int32_t cand[kChunk];
    int32_t wv[kChunk];               // value written by draw t (moved into position p_t)
    int16_t sidx[kChunk];
    int16_t prv[kChunk];
    int16_t ptr[kChunk];
    uint16_t preds[kChunk][kMaxPred];
    uint8_t st[kChunk];
    uint8_t npred[kChunk];
};

__global__ void __launch_bounds__(kVThreads, 1) samp_visit_kernel(SampArgs a, SampWork w, int s) {
    extern __shared__ __align__(16) unsigned char dyn[];
    __shared__ VisitSmem vs;
    __shared__ int warp_tot[32];
    __shared__ int s_und, s_acc;
    const int64_t b = blockIdx.x;
    SampState st = w.st[b];
    if (st.done || st.seg != s) return;
    const int tid = threadIdx.x;
    const int64_t N = a.N;
    int32_t* pool = a.use_smem ? reinterpret_cast<int32_t*>(dyn) : w.gpool + b * N;
    uint16_t* rank = a.use_smem ? reinterpret_cast<uint16_t*>(dyn + sizeof(int32_t) * N) : w.grank + b * N;
    int64_t* out = a.out_idx + b * a.ld_out;
    const uint32_t* av = w.avail + b * w.W;
    const int32_t* adj = w.adj + b * N * kAdj;
    const uint8_t* adjcnt = w.adjcnt + b * N;
    const int lvl = a.seg_level_rows[s];
    const int32_t* cnt_row = a.counts + (b * a.L + lvl) * N;
    const int64_t* indptr = a.indptr + b * (N + 1);
    const int32_t* nbr_all = a.nbr + b * a.cap_entries;
    const bool tdbg = a.dbg && b == 0 && tid == 0;
    long long tl = tdbg ? clock64() : 0;
#define VT(k)                                              \
    do {                                                   \
        if (tdbg) {                                        \
            const long long n_ = clock64();                \
            a.dbg[k] += n_ - tl;                           \
            tl = n_;                                       \
        }                                                  \
    } while (0)

    // pool = available points in index order (_kernels.py:293-298); rank table empty
    for (int64_t j = tid; j < N; j += kVThreads) rank[j] = kNoRank;
    int64_t carry = 0;
    for (int64_t base = 0; base < w.W; base += kVThreads) {
        const int64_t wd = base + tid;
        const uint32_t word = wd < w.W ? av[wd] : 0u;
        int tot;
        const int ex = block_scan(__popc(word), warp_tot, &tot);
        int64_t p = carry + ex;
        uint32_t x = word;
        while (x) {
            const int bt = __ffs(x) - 1;
            x &= x - 1;
            pool[p++] = (int32_t)(wd * 32 + bt);
        }
        carry += tot;
    }
    const int64_t L = carry;
    __syncthreads();
    VT(0);

    const uint64_t state0 = st.rng;
    const int64_t i_start = st.i;
    int64_t i = st.i;
    int64_t k = 0;
    bool ended = false;  // boundary reached inside this visit
    int64_t last_draw = -1;
    while (k < L) {
        const int K = (int)((L - k) < kChunk ? (L - k) : kChunk);
        const int64_t m0 = L - k;  // pool length before draw k
        // ---- candidate order for draws k .. k+K-1 --------------------------------
        if (a.pick_lowest) {
            if (tid < K) vs.cand[tid] = pool[k + tid];
        } else {
            // positions, then sort (position, draw)
            if (tid < K) {
                const uint64_t z = mix64v(state0 + (uint64_t)(k + tid + 1) * kGolden3);
                const uint32_t p = (uint32_t)(z % (uint64_t)(m0 - tid));
                vs.pos[tid] = p;
                vs.keys[tid] = ((unsigned long long)p << 32) | (unsigned)tid;
            } else {
                vs.keys[tid] = ~0ull;
            }
            __syncthreads();
            VT(1);
            for (int kk = 2; kk <= kChunk; kk <<= 1) {
                for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                    const int ix = tid;
                    const int px = ix ^ jj;
                    if (px > ix) {
                        const unsigned long long x0 = vs.keys[ix], x1 = vs.keys[px];
                        const bool up = (ix & kk) == 0;
                        if ((x0 > x1) == up) { vs.keys[ix] = x1; vs.keys[px] = x0; }
                    }
                    __syncthreads();
                }
            }
            if (tid < K) vs.sidx[(unsigned)vs.keys[tid]] = (int16_t)tid;
            __syncthreads();
            VT(2);
            if (tid < K) {
                const int t = tid;
                const uint32_t p = vs.pos[t];
                const int si = vs.sidx[t];
                // latest earlier draw at the same position
                int pv = -1;
                if (si > 0 && (uint32_t)(vs.keys[si - 1] >> 32) == p) pv = (int)(unsigned)vs.keys[si - 1];
                vs.prv[t] = (int16_t)pv;
                // latest earlier draw that wrote position last_t = m0 - 1 - t
                const unsigned long long target = ((unsigned long long)(uint32_t)(m0 - 1 - t) << 32) | (unsigned)t;
                int lo = 0, hi = K;  // first index with key >= target
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (vs.keys[mid] < target) lo = mid + 1; else hi = mid;
                }
                int wl = -1;
                if (lo > 0 && (uint32_t)(vs.keys[lo - 1] >> 32) == (uint32_t)(m0 - 1 - t))
                    wl = (int)(unsigned)vs.keys[lo - 1];
                vs.ptr[t] = (int16_t)(wl >= 0 ? wl : t);
            }
            __syncthreads();
            VT(3);
            // pointer jumping to the chain root (a draw whose last slot was untouched)
            for (int r = 0; r < 11; ++r) {
                int16_t np = 0;
                if (tid < K) np = vs.ptr[vs.ptr[tid]];
                __syncthreads();
                if (tid < K) vs.ptr[tid] = np;
                __syncthreads();
            }
            if (tid < K) vs.wv[tid] = pool[m0 - 1 - vs.ptr[tid]];
            __syncthreads();
            VT(4);
            if (tid < K) {
                const int pv = vs.prv[tid];
                vs.cand[tid] = pv >= 0 ? vs.wv[pv] : pool[vs.pos[tid]];
            }
            __syncthreads();
            // live positions keep the value of their last write
            if (tid < K) {
                const unsigned long long kx = vs.keys[tid];
                const uint32_t p = (uint32_t)(kx >> 32);
                const bool lastw = (tid == K - 1) || (uint32_t)(vs.keys[tid + 1] >> 32) != p;
                if (lastw && (int64_t)p < m0 - K) pool[p] = vs.wv[(unsigned)kx];
            }
        }
        __syncthreads();
        VT(5);
        // ---- greedy MIS over the chunk -------------------------------------------------
        const int32_t cme = tid < K ? vs.cand[tid] : 0;
        if (tid < K) {
            vs.st[tid] = kUnd;
            rank[cme] = (uint16_t)tid;
        }
        if (tid == 0) s_und = 0;
        __syncthreads();
        int und = 0;
        if (tid < K) {
            const int t = tid;
            const uint8_t nc = adjcnt[cme];
            int np = 0;
            bool outf = false, blocked = false;
            auto visit = [&](int32_t q) {
                const uint32_t rq = rank[q];
                if (rq == kAccMark) {
                    outf = true;
                } else if (rq < (uint32_t)t) {
                    const uint8_t sq = vs.st[rq];
                    if (sq == kIn) {
                        outf = true;
                    } else if (sq == kUnd) {
                        if (np < kMaxPred) vs.preds[t][np] = (uint16_t)rq;
                        ++np;
                        blocked = true;
                    }
                }
            };
            if (nc != kAdjOverflow) {
                const int4* ap = reinterpret_cast<const int4*>(adj + (int64_t)cme * kAdj);
                int4 v4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v4[q] = (4 * q < nc) ? __ldg(ap + q) : make_int4(0, 0, 0, 0);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    if (q < nc) {
                        const int4 x4 = v4[q >> 2];
                        visit((q & 3) == 0 ? x4.x : (q & 3) == 1 ? x4.y : (q & 3) == 2 ? x4.z : x4.w);
                    }
                }
            } else {
                const int32_t m = cnt_row[cme];
                const int32_t* row = nbr_all + indptr[cme];
                for (int32_t u = 0; u < m; ++u) {
                    const int32_t q = __ldg(row + u);
                    if (q != cme) visit(q);
                }
            }
            vs.npred[t] = np > kMaxPred ? kPredOverflow : (uint8_t)np;
            if (outf) vs.st[t] = kOut;
            else if (!blocked) vs.st[t] = kIn;
            else und = 1;
        }
        und = __reduce_add_sync(kFull, und);
        if ((tid & 31) == 0 && und) atomicAdd(&s_und, und);
        __syncthreads();
        VT(6);
        while (s_und != 0) {
            __syncthreads();
            if (tid == 0) s_und = 0;
            __syncthreads();
            int u2 = 0;
            if (tid < K && vs.st[tid] == kUnd) {
                const int t = tid;
                bool outf = false, blocked = false;
                const uint8_t np = vs.npred[t];
                if (np != kPredOverflow) {
                    for (int j = 0; j < np; ++j) {
                        const uint8_t sq = vs.st[vs.preds[t][j]];
                        if (sq == kIn) { outf = true; break; }
                        if (sq == kUnd) blocked = true;
                    }
                } else {
                    auto check = [&](int32_t q) {
                        const uint32_t rq = rank[q];
                        if (rq == kAccMark) { outf = true; return; }
                        if (rq < (uint32_t)t) {
                            const uint8_t sq = vs.st[rq];
                            if (sq == kIn) outf = true;
                            else if (sq == kUnd) blocked = true;
                        }
                    };
                    const uint8_t nc = adjcnt[cme];
                    if (nc != kAdjOverflow) {
                        for (int q = 0; q < nc && !outf; ++q) check(adj[(int64_t)cme * kAdj + q]);
                    } else {
                        const int32_t m = cnt_row[cme];
                        const int32_t* row = nbr_all + indptr[cme];
                        for (int32_t u = 0; u < m && !outf; ++u) {
                            const int32_t q = row[u];
                            if (q != cme) check(q);
                        }
                    }
                }
                if (outf) vs.st[t] = kOut;
                else if (!blocked) vs.st[t] = kIn;
                else u2 = 1;
            }
            u2 = __reduce_add_sync(kFull, u2);
            if ((tid & 31) == 0 && u2) atomicAdd(&s_und, u2);
            __syncthreads();
        }
        VT(7);
        if (tdbg) a.dbg[11] += 1;
        // ---- ordered compaction; truncation at the boundary -----------------------------
        const int64_t need = a.boundaries[st.seg] - i;
        const int flag = (tid < K && vs.st[tid] == kIn) ? 1 : 0;
        int tot;
        const int ex = block_scan(flag, warp_tot, &tot);
        const int64_t take = (int64_t)tot < need ? (int64_t)tot : need;
        const bool ends = take == need;
        if (flag && ex < take) {
            out[i + ex] = cme;
            if (ex == take - 1 && ends) s_acc = tid;
        }
        if (tid < K) rank[cme] = kNoRank;
        __syncthreads();
        if (!ends)
            for (int64_t x = tid; x < take; x += kVThreads) rank[out[i + x]] = kAccMark;
        else
            last_draw = k + s_acc;
        i += take;
        __syncthreads();
        VT(8);
        if (ends) { ended = true; break; }
        k += K;
    }

    // accepted points join the taken set; reset the accepted marks
    uint32_t* tk = w.taken + b * w.W;
    for (int64_t x = i_start + tid; x < i; x += kVThreads) {
        const int32_t p = (int32_t)out[x];
        atomicOr(&tk[p >> 5], 1u << (p & 31));
        if (!a.use_smem) rank[p] = kNoRank;
    }
    if (tid == 0) {
        // segment / entered / exhausted / RNG bookkeeping of _kernels.py:303-351
        st.i = i;
        if (ended) {
            if (!a.pick_lowest) st.rng = state0 + (uint64_t)(last_draw + 1) * kGolden3;
            if (i >= a.n_total) {
                st.done = 1;
            } else {
                int sg = st.seg;
                while (i >= a.boundaries[sg]) ++sg;
                st.seg = sg;
                st.entered += 1;
            }
        } else {
            // pool exhausted (_kernels.py:335-347)
            if (!a.pick_lowest) st.rng = state0 + (uint64_t)L * kGolden3;
            st.seg += 1;
            if (st.seg >= a.nseg) {
                st.exhausted = 1;
                st.done = 1;
            } else {
                st.entered += 1;
                if (i >= a.boundaries[st.seg]) {
                    int sg = st.seg;
                    while (i >= a.boundaries[sg]) ++sg;
                    st.seg = sg;
                    st.entered += 1;
                }
            }
        }
        w.st[b] = st;
    }
    VT(9);
#undef VT
}

}  // namespace

size_t sampler_ws_bytes(int64_t N, int nseg) {
    (void)nseg;
    // big per-cloud tables when they fit in shared memory: pool + rank
    const size_t smem = sizeof(int32_t) * N + sizeof(uint16_t) * N;
    return (smem + 255) & ~size_t(255);
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t sampler_v3_ws_bytes(int64_t B, int64_t N, bool big) {
    const int64_t W = (N + 31) >> 5;
    size_t s = align256(sizeof(SampState) * B);
    s += align256(sizeof(uint32_t) * B * W) * 2;
    s += align256(sizeof(int32_t) * B * N * kAdj);
    s += align256(sizeof(uint8_t) * B * N);
    if (big) s += align256(sizeof(int32_t) * B * N) + align256(sizeof(uint16_t) * B * N);
    return s;
}

cudaError_t launch_sampler_v3(SampArgs a, int64_t B, cudaStream_t s) {
    SampWork w = {};
    w.W = (a.N + 31) >> 5;
    unsigned char* p = a.gws;
    w.st = reinterpret_cast<SampState*>(p); p += align256(sizeof(SampState) * B);
    w.taken = reinterpret_cast<uint32_t*>(p); p += align256(sizeof(uint32_t) * B * w.W);
    w.avail = reinterpret_cast<uint32_t*>(p); p += align256(sizeof(uint32_t) * B * w.W);
    w.adj = reinterpret_cast<int32_t*>(p); p += align256(sizeof(int32_t) * B * a.N * kAdj);
    w.adjcnt = reinterpret_cast<uint8_t*>(p); p += align256(sizeof(uint8_t) * B * a.N);
    if (!a.use_smem) {
        w.gpool = reinterpret_cast<int32_t*>(p); p += align256(sizeof(int32_t) * B * a.N);
        w.grank = reinterpret_cast<uint16_t*>(p);
    }
    a.B = B;
    a.dbg = nullptr;
    if (getenv("PS_SAMPLER_TIMING")) {  // development aid (synchronises)
        static long long* dbg = nullptr;
        if (!dbg) cudaMalloc(&dbg, sizeof(long long) * 16);
        cudaMemsetAsync(dbg, 0, sizeof(long long) * 16, s);
        a.dbg = dbg;
    }
    const size_t dsm = a.use_smem ? sampler_ws_bytes(a.N, a.nseg) : 0;
    if (a.use_smem) {
        cudaError_t e = cudaFuncSetAttribute(samp_visit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
        if (e != cudaSuccess) return e;
    }
    samp_init_kernel<<<(unsigned)B, 256, 0, s>>>(a, w);
    const unsigned ga = (unsigned)std::min<int64_t>(148 * 16, (B * w.W + 7) / 8 + 1);
    const unsigned gj = (unsigned)std::min<int64_t>(148 * 16, (B * a.N + 255) / 256 + 1);
    for (int sg = 0; sg < a.nseg; ++sg) {
        samp_avail_kernel<<<ga, 256, 0, s>>>(a, w, sg);
        samp_adj_kernel<<<gj, 256, 0, s>>>(a, w, sg);
        samp_visit_kernel<<<(unsigned)B, kVThreads, dsm, s>>>(a, w, sg);
    }
    samp_final_kernel<<<(unsigned)((B + 127) / 128), 128, 0, s>>>(a, w);
    if (a.dbg) {
        long long h[16];
        cudaMemcpyAsync(h, a.dbg, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "[visit timing] cycles: pool %lld positions %lld sort %lld links %lld jump+wv %lld "
                "cand %lld mis0 %lld rounds %lld compact %lld final %lld chunks %lld\n", h[0], h[1], h[2], h[3],
                h[4], h[5], h[6], h[7], h[8], h[9], h[11]);
    }
    return cudaGetLastError();
}

size_t sampler_global_ws_bytes(int64_t B, int64_t N, bool big) {
    const size_t a = sampler_v3_ws_bytes(B, N, big), b = sampler_v4_ws_bytes(B, N);
    return a > b ? a : b;
}

// v4 (one persistent cluster kernel per batch, sampler_v4.cu) unless
// PS_SAMPLER=3 selects this per-segment kernel sequence
cudaError_t launch_sampler(SampArgs a, int64_t B, cudaStream_t s) {
    const char* e = getenv("PS_SAMPLER");
    if (e && atoi(e) == 3) return launch_sampler_v3(a, B, s);
    return launch_sampler_v4(a, B, s);
}

}  // namespace ps
