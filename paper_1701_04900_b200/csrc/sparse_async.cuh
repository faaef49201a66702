// sparse_async.cuh -- asynchronous scalar-block updates on a CSC matrix.
//
// Algorithm 1 [PAPER.md:246-260] with N = n scalar blocks (the paper's own setting,
// "always setting N=n" [PAPER.md:382]).  Persistent warps are the asynchronous workers.
// Work is handed out in BATCHES of BS consecutive sequence numbers of one epoch (a batch
// never crosses an epoch boundary, so it never holds the same block twice): batch t is
// epoch e = t / NB, positions [i0, i0 + BS) with i0 = (t mod NB) BS, NB = ceil(N / BS).
// Each batch is claimed by one warp from a global atomic counter; LPC lanes per column,
// so BS = 32 / LPC block updates are in flight per warp at once (the update's chain is a
// few dependent L2 round trips -- colptr, row indices, the residual gathers -- so the
// warp keeps many independent chains in flight instead of one).  Per update: gather the
// column's nonzeros, read the shared residual at those rows (inconsistent read),
// phi'(r) . a_j, the closed-form best response (Eq. 2), (S.4) on x_j, and scatter
// a_j dx_j back into r with red.add.
//
// Guards (checked for the whole batch before it reads; all point to strictly older
// batches, so co-resident warps cannot deadlock):
//   * bounded delay D1 [PAPER.md:224] through window counters: batches are grouped in windows
//     of W consecutive batches; the warp that completes batch t adds 1 to wcnt[(t / W) mod S]
//     (monotone: window w is complete when its slot holds (w / S + 1) W).  Batch t reads only
//     when every window that holds a batch up to batch(k_max(t) - delta - 1) is complete (all
//     such batches applied, so D1 holds exactly).  No warp ever walks a global watermark: each
//     warp keeps its own count of leading complete windows and advances it 32 windows per
//     L2 round trip (one counter per lane, ballot).  The host picks W <= ceil((delta + 2) / BS) - 1,
//     so those windows end strictly before batch t, and S > (delta + 2) / W + 2, so a slot
//     is reused only after its previous window is complete;
//   * own-block freshness D4 [PAPER.md:233]: ver[j] = number of applied updates of block j;
//     the update of epoch e waits for ver[j] >= e.  With the cyclic schedule and delta < N the
//     block's previous update (sequence k - N) is among the sequences D1 already waits for, so
//     ver[] is neither read nor written (use_ver = 0: two L2 operations per update less).
// delta == 0 gives BS = W = 1 and the sequential (d^k = 0) scheme, bit-reproducible.
// Observed delay: sampled on every 32nd batch of a warp, after a refresh of its window count wm:
// the largest k - k_first(W * wm) over the batch's sequences at read time (an upper bound on d^k
// of Assumption D1 at that read: every update before batch W * wm was applied).
#pragma once
#include "common.cuh"

namespace asy {

struct SparseAsyncParams {
    const int64_t* __restrict__ colptr;
    const int32_t* __restrict__ rowidx;
    const double* __restrict__ vals;
    int64_t m, n;
    double* r;         // the residual's pair buffer [r_i, aux_i] (2 m doubles; r_i at 2 i)
    double* x;
    const double* tau;
    Scalars S;
    double gamma;
    int sched;
    uint64_t seed;
    int64_t epoch0;
    int64_t T;        // batches in this launch = sweeps * NB
    int64_t NB;       // batches per epoch
    int BS;           // block updates per batch (<= 32 / LPC, <= delay + 1)
    int64_t delay;
    unsigned long long* counter;  // batch claims
    unsigned* ver;                // [n]
    unsigned* wcnt;               // [S] completed batches of window w at slot w mod S (monotone)
    int lgW;                      // W = 2^lgW batches per window
    int lgS;                      // S = 2^lgS window slots
    unsigned* dobs;               // observed delay (max)
    int measure_delay;            // sample the observed delay (asy_tuning.measure_delay)
    int use_ver;                  // 0: D4 is implied by D1 (cyclic schedule, delay < N): ver[] is not touched
};

__device__ __forceinline__ unsigned ld_relaxed_u32_g(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32_g(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ long long ld_relaxed_s64_g(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64_g(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_s64_g(long long* p, long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_u32_g(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_add_f64_g(double* p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double2 ld_relaxed_f64x2(const double* p) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}

// residual and b / y interleaved for the launch (one 16-byte gather per nonzero), and back
__global__ void sparse_pair_pack(const double* r, const double* aux, double* ry, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        ry[2 * i] = r[i];
        ry[2 * i + 1] = aux[i];
    }
}
__global__ void sparse_pair_unpack(const double* ry, double* r, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = ry[2 * i];
}

__global__ void sparse_async_init(SparseAsyncParams P) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) {
        *P.counter = 0ull;
        *P.dobs = 0u;
    }
    for (int64_t s = tid; s < ((int64_t)1 << P.lgS); s += nth) P.wcnt[s] = 0u;
    for (int64_t j = tid; j < P.n; j += nth) P.ver[j] = 0u;
}

#ifndef ASY_SPARSE_THREADS
#define ASY_SPARSE_THREADS 128
#endif
#ifndef ASY_SPARSE_CH
#define ASY_SPARSE_CH 8  // nonzeros per lane held in registers (longer columns loop over the rest)
#endif
#ifndef ASY_SPARSE_CLAIM
#define ASY_SPARSE_CLAIM 1  // batches claimed per atomic
#endif
#ifndef ASY_SPARSE_MINB
#define ASY_SPARSE_MINB 5  // resident CTAs per SM the register allocation must allow (5: <= 102 registers, 20 warps)
#endif
#ifndef ASY_SPARSE_RELOAD
#define ASY_SPARSE_RELOAD 0
#endif
constexpr int kSparseThreads = ASY_SPARSE_THREADS;
constexpr int kSparseClaim = ASY_SPARSE_CLAIM;
constexpr int kSparseCh = ASY_SPARSE_CH;

// LPC lanes per column (1, 2, 4 or 8): batch lanes b = lane / LPC, element lane e = lane % LPC.
template <int LOSS, int LPC>
__global__ void __launch_bounds__(kSparseThreads, ASY_SPARSE_MINB) sparse_async_kernel(SparseAsyncParams P) {
    const int lane = threadIdx.x & 31;
    const int bl = lane / LPC, el = lane % LPC;
    const unsigned cmask = LPC == 32 ? 0xffffffffu : (((1u << LPC) - 1u) << (bl * LPC));
    const int64_t N = P.n, NB = P.NB;
    const int BS = P.BS;
    const int half = perm_half_bits(N);
    const int lgW = P.lgW, lgS = P.lgS;
    const long long Smask = (1ll << lgS) - 1;
    long long wmw = 0;  // this warp's count of leading complete windows (warp-uniform)
    unsigned iter = 0;
    PermKeys pk{};
    int64_t pkE = -1;
    unsigned dmax = 0;

    // the head of a batch's update for this lane: sequence, block, column extent, tau, ver.
    // ver is read with ld.acquire: when it shows the block's previous update applied (D4), every
    // later read of this warp sees that update's writes.
    struct Head {
        long long t;      // batch
        int64_t e, k, j;  // epoch (local), sequence (local), block = column
        int64_t s, s1;    // column extent [s, s1)
        bool live;        // this lane's update exists
        unsigned vj;
        double tj;
    };
    auto head = [&](long long t) {
        Head h;
        h.t = t;
        h.e = t / NB;
        const int64_t i0 = (t - h.e * NB) * (int64_t)BS;
        const int64_t i = i0 + bl;
        h.live = t < P.T && bl < BS && i < N;
        h.k = h.e * N + i;
        h.j = 0; h.s = 0; h.s1 = 0; h.vj = 0; h.tj = 1.0;
        if (h.live) {
            h.j = i;
            if (P.sched == SCHED_RANDOM) {
                const int64_t E = P.epoch0 + h.e;
                if (E != pkE) { pk = perm_keys(P.seed, E); pkE = E; }
                uint64_t v = (uint64_t)i;
                do { v = feistel(v, half, pk); } while (v >= (uint64_t)N);
                h.j = (int64_t)v;
            }
            h.s = __ldg(&P.colptr[h.j]);
            h.s1 = __ldg(&P.colptr[h.j + 1]);
            if (el == 0) {
                if (P.use_ver) h.vj = ld_acquire_u32_g(&P.ver[h.j]);
                h.tj = __ldg(&P.tau[h.j]);
            }
        }
        return h;
    };
    auto kfirst = [&](long long t) { const int64_t e = t / NB; return e * N + (t - e * NB) * (int64_t)BS; };
    // batch containing sequence k (local numbering)
    auto batch_of = [&](long long k) { const int64_t e = k / N; return e * NB + (k - e * N) / BS; };

    // Completion of a batch: fence (every lane's r red.adds and x store of the batch first), then
    // the per-block versions and one count on the batch's window.  It is issued one iteration
    // late -- after the next batch's gathers, when the batch's writes have long reached L2 and
    // the fence costs little -- except that a warp never waits in a guard while holding one.
    long long pend = -1;
    int64_t pend_j = 0;
    bool pend_live = false;
    auto release = [&]() {
        if (pend < 0) return;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        __syncwarp();
        if (P.use_ver && pend_live && el == 0) red_relaxed_u32_g(&P.ver[pend_j], 1u);
        if (lane == 0) red_relaxed_u32_g(&P.wcnt[(pend >> lgW) & Smask], 1u);
        pend = -1;
    };

    // claims run one batch ahead: the atomic for the batch after the next one is in flight
    // while the current batch runs; each atomic claims kSparseClaim consecutive batches
    long long t0 = 0;
    if (lane == 0) t0 = (long long)atomicAdd(P.counter, (unsigned long long)kSparseClaim);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    Head cur = head(t0);
    long long cbase = t0;
    int cused = 1;
    unsigned long long cl = 0;
    if (kSparseClaim == 1 && lane == 0) cl = atomicAdd(P.counter, 1ull);
    while (cur.t < P.T) {
        long long tn;
        if (kSparseClaim == 1) {
            tn = __shfl_sync(0xffffffffu, (long long)cl, 0);
            if (lane == 0) cl = atomicAdd(P.counter, 1ull);
        } else {
            if (cused == kSparseClaim) {
                tn = __shfl_sync(0xffffffffu, (long long)cl, 0);
                cbase = tn;
                cused = 1;
            } else {
                tn = cbase + cused++;
                // the next claim goes out with the group's last batch
                if (cused == kSparseClaim && lane == 0) cl = atomicAdd(P.counter, (unsigned long long)kSparseClaim);
            }
        }
        const Head nx = head(tn);
        // D1: every window holding a batch up to batch(k_max - delta - 1) complete
        const int64_t i0 = (cur.t - cur.e * NB) * (int64_t)BS;
        const int64_t nlive = (N - i0) < BS ? (N - i0) : BS;
        const long long kd = cur.e * N + i0 + nlive - 1 - P.delay - 1;
        const long long nw = kd >= 0 ? (batch_of(kd) + (1ll << lgW)) >> lgW : 0;  // windows needed
        // D4: the previous update of this block applied
        const bool d4 = P.use_ver && cur.live && el == 0 && cur.vj < (unsigned)cur.e;
        const bool d4any = __any_sync(0xffffffffu, d4);
        if (wmw < nw || d4any) release();
        // every 32nd batch of a warp refreshes its window count even when the guard holds (the
        // observed delay below is then the real lag of the residual, not of a stale count)
        const bool sample = P.measure_delay && (++iter & 31) == 0;
        if (wmw < nw || sample) {
            unsigned ns = 32;
            for (;;) {
                // lane l: is window wmw + l complete?
                const long long w = wmw + lane;
                const unsigned c = ld_acquire_u32_g(&P.wcnt[w & Smask]);
                const bool ok = c >= (unsigned)(((w >> lgS) + 1) << lgW);
                const unsigned bal = __ballot_sync(0xffffffffu, ok);
                wmw += bal == 0xffffffffu ? 32 : __ffs(~bal) - 1;
                if (bal == 0xffffffffu) continue;  // maybe more complete windows
                if (wmw >= nw) break;
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
            }
        }
        // observed delay: sequences before batch W * wmw are all applied
        if (sample && cur.live && el == 0) {
            const long long miss = cur.k - kfirst(wmw << lgW);
            if (miss > (long long)dmax) dmax = (unsigned)miss;
        }
        if (d4) {
            unsigned ns = 32;
            while (ld_acquire_u32_g(&P.ver[cur.j]) < (unsigned)cur.e) {
                __nanosleep(ns);
                if (ns < 256) ns <<= 1;
            }
        }
        __syncwarp();  // every lane's reads below are ordered after the guards' acquire loads
        double d = 0.0, xn = 0.0;
        int32_t rows[kSparseCh];
        double vv[kSparseCh];
        const int64_t cnt = cur.s1 - cur.s;
        if (cur.live) {
            double xj = 0.0;
            if (el == 0) xj = ld_relaxed_f64(&P.x[cur.j]);
            // gradient: sum_q a_qj phi'(r_q) over the column (inconsistent read of r)
#pragma unroll
            for (int u = 0; u < kSparseCh; ++u) {
                const int64_t q = el + (int64_t)u * LPC;
                rows[u] = 0;
                vv[u] = 0.0;
                if (q < cnt) {
                    rows[u] = __ldg(&P.rowidx[cur.s + q]);
                    vv[u] = __ldg(&P.vals[cur.s + q]);
                }
            }
            double acc = 0.0;
#pragma unroll
            for (int u = 0; u < kSparseCh; ++u) {
                const int64_t q = el + (int64_t)u * LPC;
                if (q < cnt) {
                    const double2 ra = ld_relaxed_f64x2(&P.r[2 * (int64_t)rows[u]]);
                    acc = fma(vv[u], loss_prime_t<LOSS>(P.S, ra.x, ra.y), acc);
                }
            }
            for (int64_t q = el + (int64_t)kSparseCh * LPC; q < cnt; q += LPC) {
                const int32_t row = __ldg(&P.rowidx[cur.s + q]);
                const double2 ra = ld_relaxed_f64x2(&P.r[2 * (int64_t)row]);
                acc = fma(__ldg(&P.vals[cur.s + q]), loss_prime_t<LOSS>(P.S, ra.x, ra.y), acc);
            }
#pragma unroll
            for (int o = LPC / 2; o >= 1; o >>= 1) acc += __shfl_xor_sync(cmask, acc, o);
            if (el == 0) {
                const double xh = best_response(P.S, acc, xj, cur.tj, cur.j);
                xn = xj + P.gamma * (xh - xj);
                d = xn - xj;
            }
            if (LPC > 1) d = __shfl_sync(cmask, d, bl * LPC);
        }
        // the previous batch's completion, then this batch's writes
        release();
        if (cur.live) {
            if (el == 0) P.x[cur.j] = xn;
            if (d != 0.0) {
#pragma unroll
                for (int u = 0; u < kSparseCh; ++u) {
                    const int64_t q = el + (int64_t)u * LPC;
#if ASY_SPARSE_RELOAD
                    // (values and rows re-read at scatter time -- L1 / L2 hits -- instead of held in
                    // registers across the gathers: 24 registers less, one more resident CTA per SM)
                    if (q < cnt)
                        red_relaxed_add_f64_g(&P.r[2 * (int64_t)__ldg(&P.rowidx[cur.s + q])], __ldg(&P.vals[cur.s + q]) * d);
#else
                    if (q < cnt) red_relaxed_add_f64_g(&P.r[2 * (int64_t)rows[u]], vv[u] * d);
#endif
                }
                for (int64_t q = el + (int64_t)kSparseCh * LPC; q < cnt; q += LPC)
                    red_relaxed_add_f64_g(&P.r[2 * (int64_t)__ldg(&P.rowidx[cur.s + q])], __ldg(&P.vals[cur.s + q]) * d);
            }
        }
        pend = cur.t;
        pend_j = cur.j;
        pend_live = cur.live;
        cur = nx;
    }
    release();
    // warp max of the observed delay, one atomic per warp
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned v = __shfl_xor_sync(0xffffffffu, dmax, o);
        dmax = v > dmax ? v : dmax;
    }
    if (lane == 0 && dmax > 0) atomicMax(P.dobs, dmax);
}

}  // namespace asy
