// dense_async.cuh -- the fused asynchronous block-update kernel (dense A).
//
// Algorithm 1 [PAPER.md:246-260] on one B200.  Persistent CTAs are the
// asynchronous workers.  Work is handed out from ONE global atomic counter in
// units of "panel subtasks": subtask t = (sequence k = t / G, panel p = t % G),
// where sequence k updates block b = schedule(k) (S.1) and panel p covers
// rows [p*R, p*R+R) of that block's columns A_b: an R x B tile loaded by one
// 2-D TMA (cp.async.bulk.tensor, OOB rows/columns zero-filled) into a stage of
// a 4-deep shared-memory ring, together with the R residual rows it needs and
// the R rows of b / y (1-D bulk copies; the residual is read at issue time:
// the inconsistent read of the shared residual).
//
// Warp roles.  Four "pairs" q = 0..3; pair q owns smem stage q and the TMEM
// lane quarter [32q, 32q+32), split into two 256-column panel slots:
//   warp 13 (lane 0)  scheduler: claims subtasks in batches of P.claim (<= kClaim) from the
//                     counter, checks the guards below (acquire) and queues the
//                     admitted subtasks in shared memory;
//   warp 12 (lane 0)  producer: pops the queue, arms the stage mbarrier and
//                     issues the three bulk copies;
//   warp 4+q  (dot)   w = phi'(r) on the panel rows, A_{b,p}^T w straight from
//                     shared memory (lane = rows, 16 column accumulators,
//                     butterfly transpose-reduction), red.add into the
//                     sequence's accumulator; if the TMEM slot of the axpy warp
//                     that will take the panel is free, parks the panel there
//                     (smem -> registers -> tcgen05.st), otherwise marks it
//                     "re-read"; frees the smem stage, release-adds the
//                     sequence's arrival counter and queues a hand-off note.
//                     It never waits on TMEM or on a block's completion, so
//                     every loaded panel is published (no deadlock however many
//                     panels a block has);
//   warps q, 8+q      (axpy, alternating hand-offs of pair q): wait until all G
//                     panels of the sequence arrived, solve the block
//                     subproblem (Eq. 2, closed form) and (S.4) -- every panel
//                     of the block does it redundantly and bit-identically,
//                     writing the new x_b into the other half of a
//                     double-buffered x -- read the panel back (TMEM, or A
//                     again from L2 when it was not parked), push A_{b,p} dx_b
//                     into r (red.add), free the TMEM slot; completion
//                     (release-adds of the sequence and block counters) is
//                     issued one panel later unless the warp would block.
// No "last panel" role exists: all counters are monotonic (sequence k owns
// arrival / completion counts ((k/S)+1)*G in slot k mod S), the accumulator is
// double-buffered per slot use and zeroed by the next use's consumers, and x
// is double-buffered per epoch.
// Guards, checked by the scheduler before a panel is loaded (all point to
// strictly older sequences -> deadlock free with co-resident CTAs):
//   * D4 freshness [PAPER.md:233]: block b is not read before its previous
//     update is complete -- applied to r and written to x (xver[b] = u*G);
//   * bounded delay D1 [PAPER.md:224]: sequence k does not read before EVERY
//     sequence up to k - delay - 1 is complete.  Sequences are grouped in windows of W
//     consecutive sequences; every completed panel adds 1 to its window's counter
//     (wcnt[w mod SW], monotone), so window w is complete when it holds (w / SW + 1) W G.
//     The scheduler keeps its count of leading complete windows and admits sequence k only
//     when every window holding a sequence <= k - delay - 1 is complete (one counter load
//     per W sequences; W <= delay + 1 keeps those windows older than k);
//   * slot reuse: sequence k - S (previous user of the slot) is complete -- implied by D1
//     (S > delay + 1).
// delay == 0 makes the kernel the sequential (d^k = 0) scheme and, with the
// fixed-order partial reduction (deterministic = 1), bit-reproducible.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace asy {

constexpr int kPairs = 4;
#ifndef ASY_AXPY_PER_PAIR
#define ASY_AXPY_PER_PAIR 2
#endif
constexpr int kAxpyPerPair = ASY_AXPY_PER_PAIR;  // axpy warps per pair (2: hand-offs alternate)
constexpr int kTmemSlots = 2;        // parked panels per pair (TMEM lane quarter = 2 x 256 columns)
constexpr int kProducerWarp = kPairs * (1 + kAxpyPerPair);  // after axpy (0-3[, 8-11]) and dot (4-7)
constexpr int kSchedWarp = kProducerWarp + 1;
constexpr int kDenseThreads = 32 * (kSchedWarp + 1);
constexpr int kSlotsPerAx = 2 / kAxpyPerPair;  // TMEM slots owned by each axpy warp
#ifndef ASY_ROLL
#define ASY_ROLL 1   // unroll factor of the per-lane row loops (1: rolled, small I-cache footprint)
#endif
constexpr int kRoll = ASY_ROLL;
#ifndef ASY_QUEUE
#define ASY_QUEUE 2
#endif
#ifndef ASY_CLAIM
#define ASY_CLAIM 4  // most subtasks claimed per atomic (runtime: DenseAsyncParams::claim)
#endif
#ifndef ASY_SCHED_DUMMY
#define ASY_SCHED_DUMMY 0
#endif
constexpr int kQueue = ASY_QUEUE;    // scheduler -> producer queue depth
constexpr int kWs = 4;               // D1 window counters a sampling batch loads at once
constexpr int kRing = 32;            // hand-off notes per axpy warp
constexpr int kMaxRowsPerLane = 8;   // R <= 256 (one TMA box per panel)
constexpr int kClaim = ASY_CLAIM;    // subtasks claimed per atomic
constexpr int kSlotCols = 256;       // TMEM columns per parked panel
constexpr unsigned long long kParkWaitNs = 20000;  // max wait for a TMEM slot before re-reading
// Per-block all-reduce layout: panel p adds its partial into accumulator replica p mod
// kPanelRep (G ~ 80 panels adding into one copy serialise on a few L2 slices); the solves sum
// the replicas.  Counters polled by many warps sit one per 128-byte line (stride kCtrPad).
#ifndef ASY_PANEL_REP
#define ASY_PANEL_REP 1
#endif
#ifndef ASY_PANEL_PAD
#define ASY_PANEL_PAD 32
#endif
constexpr int kPanelRep = ASY_PANEL_REP;
constexpr int kCtrPad = ASY_PANEL_PAD;

struct DenseAsyncParams {
    const double* A;  // for re-reads of panels that were not parked in TMEM
    int64_t lda;
    int64_t m, n;
    int64_t B;      // block size
    int64_t nblk;   // number of blocks
    int64_t R;      // panel rows (multiple of 32, <= 256) = TMA box rows
    int64_t G;      // panels per block
    double* r;      // shared residual (LS: Ax-b, logistic: Ax); >= m+32 entries
    const double* aux;  // b (LS) or y (logistic); >= m+32 entries
    double* x0;     // x buffer read in even local epochs (written in odd ones)
    double* x1;     // x buffer read in odd local epochs
    const double* tau;
    Scalars S;
    double gamma;
    int sched;
    uint64_t seed;
    int64_t epoch0;   // schedule epoch of sequence 0 of this launch
    int64_t T;        // subtasks in this launch = K*G
    int64_t delay;    // bounded delay window (>= 0)
    int deterministic;
    int use_tmem;     // park panels in TMEM when they fit (cols_per_panel <= kSlotCols)
    int keep_in_l2;   // blocks too large to park: load with L2 evict_normal so re-reads hit L2
    int claim;        // subtasks claimed per atomic (1..kClaim)
    // synchronisation state (initialised by dense_async_init)
    unsigned long long* counter;
    double* gacc;        // [S][2][Bmax] accumulated A_b^T w; sequence k uses [k mod S][(k/S) & 1]
    double* part;        // [G][Bmax]  per-panel partials (deterministic mode)
    unsigned* arrive;    // [S]        monotonic: published panels of all users of the slot
    unsigned* consumed;  // [S]        monotonic: completed panels of all users of the slot
    unsigned* xver;      // [nblk]     monotonic: completed panels of all updates of block b
    int64_t slots;       // power of two
    int lg_slots;        // log2(slots)
    int32_t Bmax;        // = B
    int32_t Bpad;        // B rounded up to 8 (TMEM row layout)
    unsigned* wcnt;      // [SW]       monotonic: completed panels of the windows using the slot (D1)
    int lg_w;            // log2 W (sequences per window)
    int lg_sw;           // log2 SW (window slots)
    int measure_delay;   // sample the observed delay (costs scheduler stalls; asy_tuning.measure_delay)
    unsigned* dobs;      // observed delay: max over sampled admissions of k - W * (leading complete windows)
    unsigned long long* prof;   // optional [grid][warps][8] clock64 segment sums (debug; null = off)
    unsigned long long* trace;  // optional [trace_n][8] globaltimer stamps (debug; null = off)
    int64_t trace_n;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define ASY_TRACE(P_, t_, slot_)                                                   \
    do {                                                                           \
        if ((P_).trace && (t_) >= 0 && (t_) < (P_).trace_n && lane == 0)           \
            (P_).trace[(t_) * 12 + (slot_)] = gtimer();                             \
    } while (0)

struct StageMeta {
    long long t, k, b, p;
    long long u;  // local epoch of sequence k (k / N): x double buffer, D4 guard
};

// clock64 segment profiler (debug): seg[i] += cycles since the previous mark
// (compiled in only with -DASY_SEGPROF -- a profiling build, `build.py --variant prof
// ASY_SEGPROF`, loaded with ASY_LIB_VARIANT=prof; otherwise every call is empty)
struct SegProf {
#ifdef ASY_SEGPROF
    unsigned long long seg[8];
    long long last;
    __device__ void start() {
        for (int i = 0; i < 8; ++i) seg[i] = 0;
        last = clock64();
    }
    __device__ void mark(int i) {
        const long long t = clock64();
        seg[i] += (unsigned long long)(t - last);
        last = t;
    }
    __device__ void flush(unsigned long long* out, int lane) {
        if (out && lane == 0)
            for (int i = 0; i < 8; ++i) out[i] = seg[i];
    }
#else
    __device__ void start() {}
    __device__ void mark(int) {}
    __device__ void flush(unsigned long long*, int) {}
#endif
};

struct Handoff {
    StageMeta md;
    int parked;   // 1 + TMEM slot of the parked panel; 0: re-read A from global
    int pad;
};

__global__ void dense_async_init(DenseAsyncParams P) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) *P.counter = 0ull;
    for (int64_t s = tid; s < P.slots; s += nth) {
        P.arrive[s * kCtrPad] = 0u;
        P.consumed[s * kCtrPad] = 0u;
    }
    for (int64_t i = tid; i < 2 * P.slots * kPanelRep * P.Bmax; i += nth) P.gacc[i] = 0.0;
    for (int64_t i = tid; i < P.nblk; i += nth) P.xver[i * kCtrPad] = 0u;
    for (int64_t i = tid; i < ((int64_t)1 << P.lg_sw); i += nth) P.wcnt[i * kCtrPad] = 0u;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void red_add_u32(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_u32(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acqrel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ long long ld_relaxed_s64(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
#ifndef ASY_SPIN_MIN
#define ASY_SPIN_MIN 32
#endif
#ifndef ASY_SPIN_MAX
#define ASY_SPIN_MAX 256
#endif
__device__ __forceinline__ void spin_until_ge_relaxed(const unsigned* p, unsigned v) {
    unsigned ns = ASY_SPIN_MIN;
    while (ld_relaxed_u32(p) < v) {
        __nanosleep(ns);
        if (ns < ASY_SPIN_MAX) ns <<= 1;
    }
}

// ---- TMEM (tcgen05) ---------------------------------------------------------
__device__ __forceinline__ void tmem_alloc_512(uint32_t* dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst_smem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_512(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 8 doubles (16 x b32 columns) of this thread's TMEM lane
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const double* v) {
    uint32_t u[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(v[i]);
        u[2 * i] = (uint32_t)b;
        u[2 * i + 1] = (uint32_t)(b >> 32);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};" ::"r"(taddr),
        "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]), "r"(u[8]),
        "r"(u[9]), "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]), "r"(u[15])
        : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* u) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ double u2d(uint32_t lo, uint32_t hi) {
    return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}

// Butterfly reduce-scatter over 16 columns: in: v[c] = this lane's partial of
// column c; out: lanes l and l^16 return the warp total of column l & 15.
__device__ __forceinline__ double transpose_reduce16(double (&v)[16], int lane) {
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

__device__ __forceinline__ unsigned ld_acquire_cta_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_cta_u32(unsigned* p, unsigned v) {
    asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_cta_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// Butterfly reduce-scatter over 8 columns: lanes with l & 7 == c return column c's total.
__device__ __forceinline__ double transpose_reduce8(double (&v)[8], int lane) {
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double send = up ? v[i] : v[i + o];
            const double keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    const double t = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 8);
    return t + __shfl_xor_sync(0xffffffffu, t, 16);
}

// 16 doubles of a 32 x 16 sub-tile for one lane (see the dot warps): two columns (stride ld),
// four row pairs at offsets o0, o1, 16 + o0, 16 + o1 from a.
__device__ __forceinline__ void load_subtile(const double* a, int ld, int o0, int o1, double (&v)[16]) {
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
        const double2 t0 = *reinterpret_cast<const double2*>(a + cc * ld + o0);
        const double2 t1 = *reinterpret_cast<const double2*>(a + cc * ld + o1);
        const double2 t2 = *reinterpret_cast<const double2*>(a + cc * ld + 16 + o0);
        const double2 t3 = *reinterpret_cast<const double2*>(a + cc * ld + 16 + o1);
        v[8 * cc + 0] = t0.x; v[8 * cc + 1] = t0.y;
        v[8 * cc + 2] = t1.x; v[8 * cc + 3] = t1.y;
        v[8 * cc + 4] = t2.x; v[8 * cc + 5] = t2.y;
        v[8 * cc + 6] = t3.x; v[8 * cc + 7] = t3.y;
    }
}

// BT = block width padded to a power of two >= 8 (panel columns, TMEM row layout);
// RPL = panel rows per lane (R = 32*RPL); NS = smem stages (kPairs or 2*kPairs:
// a second stage per pair overlaps the next panel's load with this one's dot).
// All compile-time so that the inner loops are fully unrolled with immediate
// shared-memory offsets.
template <int BT, int RPL, int NS, int LOSS>
__global__ void __launch_bounds__(kDenseThreads, 1)
    dense_async_kernel(const __grid_constant__ CUtensorMap tmap, const DenseAsyncParams P) {
    constexpr int NPL = (BT + 31) / 32;  // block columns per lane in the solve
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    static_assert(NS % kPairs == 0, "pair q owns stages q (mod kPairs)");
    constexpr int NAX = kPairs * kAxpyPerPair;
    constexpr int R = 32 * RPL;
    constexpr int Bpad = BT;
    constexpr int GW = BT < 16 ? BT : 16;    // column group of the dot pass
    const int Bmax = P.Bmax;
    constexpr size_t PANEL = (size_t)R * BT;  // doubles of A per stage (TMA box R x BT)
    constexpr size_t STAGE = PANEL + 2 * R;   // + the R residual rows + the R rows of b / y
    double* stages = reinterpret_cast<double*>(smem_raw);                       // NS * STAGE
    double* dxs = stages + NS * STAGE;                                          // NAX * Bpad
    StageMeta* meta = reinterpret_cast<StageMeta*>(dxs + NAX * Bpad);          // NS
    StageMeta* queue = meta + NS;                                               // kQueue
    Handoff* ring = reinterpret_cast<Handoff*>(queue + kQueue);                 // NAX * kRing
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + NAX * kRing);           // NS
    uint64_t* empty = full + NS;                                                // NS
    uint64_t* qfull = empty + NS;                                               // kQueue
    uint64_t* qempty = qfull + kQueue;                                          // kQueue
    uint64_t* rfull = qempty + kQueue;                                          // NAX * kRing
    uint64_t* rempty = rfull + NAX * kRing;                                     // NAX * kRing
    unsigned* tm_done = reinterpret_cast<unsigned*>(rempty + NAX * kRing);      // NAX
    uint32_t* tmem_base_s = tm_done + NAX;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kProducerWarp) {
        tmem_alloc_512(tmem_base_s);
        if (lane == 0) {
            for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
            for (int s = 0; s < kQueue; ++s) { mbar_init(&qfull[s], 1); mbar_init(&qempty[s], 1); }
            for (int s = 0; s < NAX * kRing; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], 1); }
            for (int s = 0; s < NAX; ++s) tm_done[s] = 0u;
            mbar_fence_init();
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_base_s;
    constexpr int cols_per_row = 2 * Bpad;  // b32 TMEM columns per panel row

    if (warp == kProducerWarp) {
        // ------------------------------------------------------------------ producer
        if (lane == 0) {
            const uint32_t box_bytes = (uint32_t)(PANEL * 8);
            const uint64_t pol = P.keep_in_l2 ? policy_evict_normal() : policy_evict_first();
            int ends = 0;
            long long qi = 0;
            for (long long it = 0;; ++it) {
                const int st = (int)(it % NS);
                if (it >= NS) mbar_wait(&empty[st], (uint32_t)(((it / NS) - 1) & 1));
                StageMeta& md = meta[st];
                StageMeta e;
                e.t = -1;
                if (ends == 0) {
                    const int qs = (int)(qi % kQueue);
                    mbar_wait(&qfull[qs], (uint32_t)((qi / kQueue) & 1));
                    e = queue[qs];
                    mbar_arrive(&qempty[qs]);
                    ++qi;
                }
                if (e.t < 0) {  // one end marker for each pair (consecutive iterations)
                    md.t = -1;
                    mbar_arrive(&full[st]);
                    if (++ends == kPairs) break;
                    continue;
                }
                md = e;
                ASY_TRACE(P, e.t, 1);
                const long long r0 = e.p * R;
                const long long nr = (P.m - r0) < R ? (P.m - r0) : R;
                const uint32_t rbytes = (uint32_t)(((nr + 1) & ~1ll) * 8);
                double* dst = stages + st * STAGE;
#ifdef ASY_DIAG_NO_RB
                // (measurement only: no residual / b rows -- the results are meaningless)
                mbar_arrive_expect_tx(&full[st], box_bytes);
                tma_load_2d(dst, &tmap, (int)r0, (int)(e.b * P.B), &full[st], pol);
#else
                // (least squares: phi'(r) = 2 s r needs no b rows -- r = Ax - b already holds them --
                // so the panel costs two bulk copies instead of three)
                constexpr uint32_t ncopy = LOSS == LOSS_LS ? 1u : 2u;
                mbar_arrive_expect_tx(&full[st], box_bytes + ncopy * rbytes);
                tma_load_2d(dst, &tmap, (int)r0, (int)(e.b * P.B), &full[st], pol);
                bulk_g2s_nohint(dst + PANEL, P.r + r0, rbytes, &full[st]);
                if constexpr (LOSS != LOSS_LS) bulk_g2s_nohint(dst + PANEL + R, P.aux + r0, rbytes, &full[st]);
#endif
            }
        }
        __syncwarp();
    } else if (warp == kSchedWarp) {
        // ------------------------------------------------------------------ scheduler
        if (lane == 0) {
            long long qi = 0;
            auto push = [&](const StageMeta& e) {
                const int qs = (int)(qi % kQueue);
                if (qi >= kQueue) mbar_wait(&qempty[qs], (uint32_t)(((qi / kQueue) - 1) & 1));
                queue[qs] = e;
                mbar_arrive(&qfull[qs]);
                ++qi;
            };
            // Per batch: claim kClaim subtasks, evaluate the schedule (once per sequence, the
            // permutation keys once per epoch), check the guards, queue them.  The next claim's
            // atomic is issued before this batch is processed so its round trip overlaps.
            const long long G = P.G, N = P.nblk;
            const int lgW = P.lg_w, lgSW = P.lg_sw;
            const long long swmask = (1ll << lgSW) - 1;
            const unsigned WG = (unsigned)G << lgW;  // completed panels of a window
            // window w complete: its slot holds (w / SW + 1) W G completions
            auto wneed = [&](long long w) { return (unsigned)((w >> lgSW) + 1) * WG; };
            long long wdone = 0;  // leading complete windows (every sequence < W wdone complete)
            long long dmax = 0;   // observed delay (sampled)
            unsigned nbatch = 0;
            bool sample = false;
            const int half = perm_half_bits(N);
            PermKeys pk{}, pkp{};
            long long ck = -1, cb = 0, cu = 0, cE = -1, cprev = -1;  // cached sequence / block / epochs
            const int nclaim = P.claim;
            long long tb = (long long)atomicAdd(P.counter, (unsigned long long)nclaim);
            while (tb < P.T) {
                const long long tn = (long long)atomicAdd(P.counter, (unsigned long long)nclaim);
                StageMeta e[kClaim];
                unsigned xv[kClaim];
                long long kprev[kClaim];
                long long k = tb / G, p = tb - k * G;
#pragma unroll
                for (int i = 0; i < kClaim; ++i) {
                    const long long t = tb + i;
                    if (i >= nclaim) {
                        e[i].t = -1; e[i].k = 0; e[i].p = 0; e[i].b = 0; e[i].u = 0;
                        continue;
                    }
                    if (k != ck) {
                        ck = k;
                        cu = k / N;
                        const long long pos = k - cu * N;
                        cb = pos;
                        cprev = k - N;  // the block's previous update (cyclic: one epoch earlier)
                        if (P.sched == SCHED_RANDOM) {
                            const long long E = P.epoch0 + cu;
                            if (E != cE) {
                                pk = perm_keys(P.seed, E);
                                if (E > 0) pkp = perm_keys(P.seed, E - 1);
                                cE = E;
                            }
                            uint64_t v = (uint64_t)pos;
                            do { v = feistel(v, half, pk); } while (v >= (uint64_t)N);
                            cb = (long long)v;
                            // its position in the previous epoch (inverse permutation, cycle-walking)
                            if (E > 0) {
                                uint64_t w = v;
                                do { w = feistel_inv(w, half, pkp); } while (w >= (uint64_t)N);
                                cprev = (cu - 1) * N + (long long)w;
                            }
                        }
                    }
                    e[i].t = t < P.T ? t : -1;
                    e[i].k = k;
                    e[i].p = p;
                    e[i].b = cb;
                    e[i].u = cu;
                    kprev[i] = cprev;
                    ASY_TRACE(P, t, 0);
                    if (++p == G) { p = 0; ++k; }
                }
                // guards.  D1 needs a window counter load only when the bound moves into a window not
                // yet known complete (once per W sequences); every 16th batch looks up to kWs windows
                // ahead so that the observed delay tracks the real lag.  D4 (the block's previous
                // update complete) is implied by D1 when that update lies in a complete window --
                // always for the cyclic schedule with delay < N - W -- and loaded otherwise.
                long long kdmax = -1;
#pragma unroll
                for (int i = 0; i < kClaim; ++i)
                    if (e[i].t >= 0) kdmax = e[i].k - P.delay - 1;
                const long long nwmax = kdmax >= 0 ? (kdmax + (1ll << lgW)) >> lgW : 0;  // windows needed
                // observed delay (measurement mode only, asy_tuning.measure_delay): every 16th batch
                // loads the counters of the next kWs windows and advances the count of complete
                // windows over them.  Off by default: those counters sit on lines under heavy atomic
                // traffic and the scheduler would stall on them (measured 9% on configs[1]).
                if (P.measure_delay && (++nbatch & 15) == 0) {
                    unsigned wcs[kWs];
#pragma unroll
                    for (int u = 0; u < kWs; ++u) wcs[u] = ld_relaxed_u32(&P.wcnt[((wdone + u) & swmask) * kCtrPad]);
                    bool run = true;
#pragma unroll
                    for (int u = 0; u < kWs; ++u) {
                        run = run && wcs[u] >= wneed(wdone);
                        if (run) ++wdone;
                    }
                    sample = true;
                }
                // D1 needs one more window: one (blocking) load, once per W sequences
                unsigned wc = 0u;
                if (wdone < nwmax) wc = ld_relaxed_u32(&P.wcnt[(wdone & swmask) * kCtrPad]);
#pragma unroll
                for (int i = 0; i < kClaim; ++i) {
                    xv[i] = 0u;
                    if (e[i].t >= 0 && kprev[i] >= (wdone << lgW))
                        xv[i] = ld_relaxed_u32(&P.xver[e[i].b * kCtrPad]);
                }
                if (wdone < nwmax && wc >= wneed(wdone)) ++wdone;
#if ASY_SCHED_DUMMY
                {   // (measurement: the round-1 scheduler's per-batch counter loads, values unused)
                    unsigned dsum = 0;
#pragma unroll
                    for (int i = 0; i < kClaim; ++i) {
                        if (e[i].t < 0) continue;
                        const long long kk = e[i].k, kd = kk - P.delay - 1;
                        dsum += ld_relaxed_u32(&P.xver[e[i].b * kCtrPad]);
                        dsum += ld_relaxed_u32(&P.consumed[(kk & (P.slots - 1)) * kCtrPad]);
                        if (kd >= 0) dsum += ld_relaxed_u32(&P.consumed[(kd & (P.slots - 1)) * kCtrPad]);
                    }
                    if (dsum == 0xFFFFFFFFu) wdone = 0;
                }
#endif
                // admit in claim order: a subtask never waits while an older one of this batch is
                // held back.  Guards are observed with relaxed loads and a fence follows only a guard
                // that had to wait: the counters were released (fence + red) by the SMs that completed
                // the updates, and what an admitted subtask reads that they wrote -- residual rows (bulk
                // copy), x and the accumulator (ld.relaxed.gpu) -- is read from L2, never through L1.
                // (A fence or ld.acquire on every admission measured 10-14% slower.)
#pragma unroll
                for (int i = 0; i < kClaim; ++i) {
                    if (e[i].t < 0) continue;
                    const long long kk = e[i].k, kd = kk - P.delay - 1;
                    const long long nw = kd >= 0 ? (kd + (1ll << lgW)) >> lgW : 0;
                    bool waited = false;
                    while (wdone < nw) {  // D1: every window holding a sequence <= kd complete
                        spin_until_ge_relaxed(&P.wcnt[(wdone & swmask) * kCtrPad], wneed(wdone));
                        ++wdone;
                        waited = true;
                    }
                    if (kprev[i] >= (wdone << lgW)) {  // D4 not implied by D1
                        const unsigned need_x = (unsigned)e[i].u * (unsigned)G;
                        if (xv[i] < need_x) {
                            spin_until_ge_relaxed(&P.xver[e[i].b * kCtrPad], need_x);
                            waited = true;
                        }
                    }
                    if (waited) fence_acqrel_gpu();
                    if (sample && i == 0 && kk - (wdone << lgW) > dmax) dmax = kk - (wdone << lgW);
                    if (i == 0) sample = false;
                    push(e[i]);
                }
                tb = tn;
            }
            StageMeta end;
            end.t = -1; end.k = end.b = end.p = end.u = 0;
            push(end);
            if (P.dobs && dmax > 0) atomicMax(P.dobs, (unsigned)dmax);
        }
        __syncwarp();
    } else if (warp >= kPairs && warp < 2 * kPairs) {
        // ------------------------------------------------------------------ dot warps
        const int q = warp - kPairs;
        const uint32_t tlane = tmem_base + ((uint32_t)(32 * q) << 16);
        static_assert(kSlotsPerAx * kAxpyPerPair == kTmemSlots, "axpy warp h owns TMEM slots h*kSlotsPerAx..");
        unsigned tm_used0 = 0u, tm_used1 = 0u;  // panels parked for the pair's axpy warp h = 0 / 1
        const int rq = lane & 3, co = lane >> 2;
        const int o0 = 8 * (co & 1), o1 = 8 - o0;  // row-pair offsets of j = 0, 1 (j = 2, 3: + 16)
        SegProf sp;
        sp.start();
        for (long long j = 0;; ++j) {
            const long long it = j * kPairs + q;  // pair q owns stage q
            const int st = (int)(it % NS);
            const int h = kAxpyPerPair == 2 ? (int)(j & 1) : 0;  // hand-offs alternate between them
            const int ax = q * kAxpyPerPair + h;                  // axpy warps of the pair
            const long long e = j / kAxpyPerPair;                 // ring position of axpy warp ax
            const int rs = (int)(e % kRing);
            Handoff* ho = &ring[ax * kRing + rs];
            uint64_t* rf = &rfull[ax * kRing + rs];
            uint64_t* re = &rempty[ax * kRing + rs];
            unsigned tm_used = h ? tm_used1 : tm_used0;
            mbar_wait(&full[st], (uint32_t)((it / NS) & 1));
            sp.mark(0);
            const StageMeta md = meta[st];
            if (md.t < 0) {
                if (lane == 0) mbar_arrive(&empty[st]);
                // end markers for both axpy warps of the pair (ring positions e and j - e)
#pragma unroll
                for (int hh = 0; hh < kAxpyPerPair; ++hh) {
                    const long long eh = hh == h ? e : (j + 1 - hh) / kAxpyPerPair;
                    const int rsh = (int)(eh % kRing);
                    const int axh = q * kAxpyPerPair + hh;
                    if (eh >= kRing) mbar_wait(&rempty[axh * kRing + rsh], (uint32_t)(((eh / kRing) - 1) & 1));
                    if (lane == 0) {
                        ring[axh * kRing + rsh].md.t = -1;
                        mbar_arrive(&rfull[axh * kRing + rsh]);
                    }
                }
                break;
            }
            const long long k = md.k, b = md.b, p = md.p;
            const long long slot = k & (P.slots - 1);
            double* gacc = P.gacc + ((slot * 2 + ((k >> P.lg_slots) & 1)) * kPanelRep + (p % kPanelRep)) * Bmax;
            const long long c0 = b * P.B;
            const int nc = (int)((P.n - c0) < P.B ? (P.n - c0) : P.B);
            const double* pan = stages + st * STAGE;
            double* rsm = stages + st * STAGE + PANEL;
            ASY_TRACE(P, md.t, 2);
            // w = phi'(r) on this lane's panel rows (residual and b / y rows arrived with the
            // panel), written over the residual rows: the row loops below stay rolled (small
            // instruction footprint) and read w back from shared memory
            const long long r0 = p * R;
#pragma unroll
            for (int qq = 0; qq < RPL; ++qq) {
                const int i = lane + 32 * qq;
                rsm[i] = (r0 + i) < P.m ? loss_prime_t<LOSS>(P.S, rsm[i], rsm[R + i]) : 0.0;
            }
            __syncwarp();  // (the dot pass reads w of other lanes' rows)
            sp.mark(1);
            // a free TMEM slot now?  then dot and park in ONE pass over shared memory
            int parked = 0;
            if (P.use_tmem) {
                unsigned ok = 0;
                if (lane == 0) ok = tm_used - ld_acquire_cta_u32(&tm_done[ax]) < (unsigned)kSlotsPerAx;
                parked = __shfl_sync(0xffffffffu, ok, 0);
                if (parked) tc_fence_after();
            }
            const int tslot_idx = h * kSlotsPerAx + (int)(tm_used % kSlotsPerAx);
            const uint32_t tslot = tlane + (uint32_t)(tslot_idx * kSlotCols);
            if constexpr (BT >= 16) {
            // Lane layout of a 32 x 16 sub-tile (rows 32 qq.., columns g0..): lane (co = lane >> 2,
            // rq = lane & 3) owns columns g0 + 2 co, + 1 and the row pairs rq + 4 (j ^ (co & 1)),
            // j < 4, read as double2 (8 conflict-free 16-byte loads per sub-tile).  The sum over
            // rows is in-lane over all RPL sub-tiles and takes two shuffles per 16 columns (a
            // lane-per-row layout needs a 16-shuffle butterfly); the axpy warps, two per dot warp,
            // pay a 7-shuffle transposing sum per 32 rows instead.
#pragma unroll
            for (int g0 = 0; g0 < BT; g0 += GW) {
                double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
#pragma unroll kRoll
                for (int qq = 0; qq < RPL; ++qq) {
                    double v[16];  // v[8 cc + 2 j + t] = A[row 32 qq + 2 (rq + 4 (j ^ par)) + t][column g0 + 2 co + cc]
                    load_subtile(pan + (size_t)(g0 + 2 * co) * R + 32 * qq + 2 * rq, R, o0, o1, v);
                    const double* wp = rsm + 32 * qq + 2 * rq;
                    const double2 w0 = *reinterpret_cast<const double2*>(wp + o0);
                    const double2 w1 = *reinterpret_cast<const double2*>(wp + o1);
                    const double2 w2 = *reinterpret_cast<const double2*>(wp + 16 + o0);
                    const double2 w3 = *reinterpret_cast<const double2*>(wp + 16 + o1);
                    a00 = fma(v[0], w0.x, a00); a01 = fma(v[1], w0.y, a01);
                    a10 = fma(v[8], w0.x, a10); a11 = fma(v[9], w0.y, a11);
                    a00 = fma(v[2], w1.x, a00); a01 = fma(v[3], w1.y, a01);
                    a10 = fma(v[10], w1.x, a10); a11 = fma(v[11], w1.y, a11);
                    a00 = fma(v[4], w2.x, a00); a01 = fma(v[5], w2.y, a01);
                    a10 = fma(v[12], w2.x, a10); a11 = fma(v[13], w2.y, a11);
                    a00 = fma(v[6], w3.x, a00); a01 = fma(v[7], w3.y, a01);
                    a10 = fma(v[14], w3.x, a10); a11 = fma(v[15], w3.y, a11);
                    if (parked) {
                        const uint32_t trow = tslot + (uint32_t)(qq * cols_per_row + 2 * g0);
                        tmem_st8(trow, v);
                        tmem_st8(trow + 16, v + 8);
                    }
                }
                // columns g0 + 2 co, + 1 summed over the four rq lanes: lanes with rq & 1 == c end
                // with column g0 + 2 co + c
                const double s0 = a00 + a01, s1 = a10 + a11;
                const bool up = (lane & 1) != 0;
                double colsum = (up ? s1 : s0) + __shfl_xor_sync(0xffffffffu, up ? s0 : s1, 1);
                colsum += __shfl_xor_sync(0xffffffffu, colsum, 2);
                const int cidx = g0 + 2 * co + rq;
                if (rq < 2 && cidx < nc) {
                    if (P.deterministic) P.part[p * Bmax + cidx] = colsum;
                    else atomicAdd(&gacc[cidx], colsum);
                }
            }
            } else {
                // (blocks of <= 8 columns: lane = row, 8-column butterfly)
#pragma unroll
            for (int g0 = 0; g0 < BT; g0 += GW) {
                double acc[GW];
#pragma unroll
                for (int c = 0; c < GW; ++c) acc[c] = 0.0;
#pragma unroll kRoll
                for (int qq = 0; qq < RPL; ++qq) {
                    const double* a = pan + (size_t)g0 * R + lane + 32 * qq;
                    const double wq = rsm[lane + 32 * qq];
                    double v[GW];
#pragma unroll
                    for (int c = 0; c < GW; ++c) v[c] = a[c * R];
#pragma unroll
                    for (int c = 0; c < GW; ++c) acc[c] = fma(v[c], wq, acc[c]);
                    if (parked) {
                        const uint32_t trow = tslot + (uint32_t)(qq * cols_per_row + 2 * g0);
#pragma unroll
                        for (int s8 = 0; s8 < GW / 8; ++s8) tmem_st8(trow + 16 * s8, v + 8 * s8);
                    }
                }
                double colsum;
                if constexpr (GW == 16) colsum = transpose_reduce16(acc, lane);
                else colsum = transpose_reduce8(acc, lane);
                if (lane < GW && g0 + lane < nc) {
                    if (P.deterministic) P.part[p * Bmax + g0 + lane] = colsum;
                    else atomicAdd(&gacc[g0 + lane], colsum);
                }
            }
            }
            ASY_TRACE(P, md.t, 3);
            sp.mark(2);
            if (!parked && P.use_tmem) {
                // no slot was free: wait a bounded time for one, then park in a second pass;
                // holding the stage indefinitely could hold back a block whose panel is queued
                // behind it, so after kParkWaitNs the panel is left in HBM/L2 (re-read later)
                unsigned ok = 0;
                if (lane == 0) {
                    const unsigned long long t0 = gtimer();
                    do {
                        __nanosleep(64);
                        ok = tm_used - ld_acquire_cta_u32(&tm_done[ax]) < (unsigned)kSlotsPerAx;
                    } while (!ok && gtimer() - t0 < kParkWaitNs);
                }
                parked = __shfl_sync(0xffffffffu, ok, 0);
                ASY_TRACE(P, md.t, 4);
                sp.mark(3);
                if (parked) {
                    tc_fence_after();
                    if constexpr (BT >= 16) {
#pragma unroll
                    for (int g0 = 0; g0 < BT; g0 += GW) {
#pragma unroll kRoll
                        for (int qq = 0; qq < RPL; ++qq) {
                            double v[16];
                            load_subtile(pan + (size_t)(g0 + 2 * co) * R + 32 * qq + 2 * rq, R, o0, o1, v);
                            const uint32_t trow = tslot + (uint32_t)(qq * cols_per_row + 2 * g0);
                            tmem_st8(trow, v);
                            tmem_st8(trow + 16, v + 8);
                        }
                    }
                    } else {
#pragma unroll
                    for (int g0 = 0; g0 < BT; g0 += GW) {
#pragma unroll kRoll
                        for (int qq = 0; qq < RPL; ++qq) {
                            const double* a = pan + (size_t)g0 * R + lane + 32 * qq;
                            double v[GW];
#pragma unroll
                            for (int c = 0; c < GW; ++c) v[c] = a[c * R];
                            const uint32_t trow = tslot + (uint32_t)(qq * cols_per_row + 2 * g0);
#pragma unroll
                            for (int s8 = 0; s8 < GW / 8; ++s8) tmem_st8(trow + 16 * s8, v + 8 * s8);
                        }
                    }
                    }
                }
            }
            if (parked) {
                if (h) ++tm_used1;
                else ++tm_used0;
                tmem_wait_st();
                tc_fence_before();
            }
            __syncwarp();
            sp.mark(4);
            // publish (the partials' red.adds drained during the parking pass)
            if (lane == 0) red_add_release_u32(&P.arrive[slot * kCtrPad], 1u);
            // hand-off note (after publishing: waiting here can never hold back a block)
            if (e >= kRing) mbar_wait(re, (uint32_t)(((e / kRing) - 1) & 1));
            if (lane == 0) {
                mbar_arrive(&empty[st]);  // smem stage free
                ho->md = md;
                ho->parked = parked ? 1 + tslot_idx : 0;
                mbar_arrive(rf);
            }
            sp.mark(5);
        }
        sp.flush(P.prof ? P.prof + ((size_t)blockIdx.x * 16 + warp) * 8 : nullptr, lane);
    } else {
        // ------------------------------------------------------------------ axpy warps
        const int q = warp & 3, h = warp / (2 * kPairs);  // warps 0-3: h = 0, warps 8-11: h = 1
        const int ax = q * kAxpyPerPair + h;
        const uint32_t tquarter = tmem_base + ((uint32_t)(32 * q) << 16);
        double* dv = dxs + ax * Bpad;
        Handoff* myring = ring + ax * kRing;
        uint64_t* myfull = rfull + ax * kRing;
        uint64_t* myempty = rempty + ax * kRing;
        unsigned tm_fin = 0;
        const int rq = lane & 3, co = lane >> 2;  // the dot warps' lane layout
        long long pend_slot = -1, pend_b = -1, pend_k = 0;  // completion of the previous panel, issued late
        auto complete = [&]() {
            if (pend_slot >= 0 && lane == 0) {
                fence_acqrel_gpu();  // r red.adds, x / accumulator writes before the counts (one membar)
                red_add_u32(&P.consumed[pend_slot * kCtrPad], 1u);
                red_add_u32(&P.xver[pend_b * kCtrPad], 1u);
                red_add_u32(&P.wcnt[((pend_k >> P.lg_w) & ((1ll << P.lg_sw) - 1)) * kCtrPad], 1u);
            }
            pend_slot = -1;
        };
        SegProf sp;
        sp.start();
        for (long long e = 0;; ++e) {
            const int rs = (int)(e % kRing);
            // the previous panel's completion is issued now unless the next one is already here;
            // never deferred across a wait (a guard elsewhere may be waiting for it)
            if (!mbar_test(&myfull[rs], (uint32_t)((e / kRing) & 1))) {
                complete();
                mbar_wait(&myfull[rs], (uint32_t)((e / kRing) & 1));
            }
            const Handoff hd = myring[rs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&myempty[rs]);
            sp.mark(0);
            const StageMeta md = hd.md;
            if (md.t < 0) break;
            const long long k = md.k, b = md.b, p = md.p;
            const long long slot = k & (P.slots - 1);
            const long long use = k >> P.lg_slots;
            const double* gacc = P.gacc + (slot * 2 + (use & 1)) * kPanelRep * Bmax;        // replica 0
            double* gnext = P.gacc + (slot * 2 + ((use + 1) & 1)) * kPanelRep * Bmax;     // replica 0
            const long long c0 = b * P.B;
            const int nc = (int)((P.n - c0) < P.B ? (P.n - c0) : P.B);
            const long long u = md.u;
            const double* xr = (u & 1) ? P.x1 : P.x0;
            double* xw = (u & 1) ? P.x0 : P.x1;
            ASY_TRACE(P, md.t, 5);
            // x_b (previous epoch, final by the D4 guard) and tau do not depend on the arrivals
            double ypre[NPL], tpre[NPL];
#pragma unroll
            for (int s4 = 0; s4 < NPL; ++s4) {
                const int c = lane + 32 * s4;
                // L2 read: another SM wrote this half of x in the previous epoch, and a line of it
                // may still sit in this SM's (non-coherent) L1 from an older epoch
                ypre[s4] = c < nc ? ld_relaxed_f64(&xr[c0 + c]) : 0.0;
                tpre[s4] = c < nc ? P.tau[c0 + c] : 1.0;
            }
            // all G partials of sequence k published?  (flush the pending completion before
            // blocking: a guard that admits this very sequence may be waiting for it)
            {
                const unsigned need = (unsigned)((use + 1) * P.G);
                unsigned ok = 0;
                // relaxed poll: everything read after it that other SMs wrote (accumulator, x) is
                // read with strong L2 loads, so no L1 invalidation (acquire) is needed
                if (lane == 0) ok = ld_relaxed_u32(&P.arrive[slot * kCtrPad]) >= need;
                ok = __shfl_sync(0xffffffffu, ok, 0);
                if (!ok) {
                    complete();
                    if (lane == 0) spin_until_ge_relaxed(&P.arrive[slot * kCtrPad], need);
                }
            }
            __syncwarp();
            ASY_TRACE(P, md.t, 6);
            sp.mark(1);
            // block subproblem (Eq. 2, closed form) + (S.4): identical in every panel of the block.
            // The accumulated gradient is loaded first; the previous panel's completion (a fence
            // that waits for its residual red.adds) is issued while those loads are in flight.
            double gv[NPL];
#pragma unroll
            for (int s4 = 0; s4 < NPL; ++s4) {
                const int c = lane + 32 * s4;
                gv[s4] = 0.0;
                if (c < nc) {
                    if (P.deterministic) {
#pragma unroll 1
                        for (long long qq = 0; qq < P.G; ++qq) gv[s4] += ld_relaxed_f64(&P.part[qq * Bmax + c]);
                    } else {
                        double gr[kPanelRep];
#pragma unroll
                        for (int r = 0; r < kPanelRep; ++r) gr[r] = ld_relaxed_f64(&gacc[r * Bmax + c]);
#pragma unroll
                        for (int r = 0; r < kPanelRep; ++r) gv[s4] += gr[r];
                    }
                }
            }
            complete();
            bool nz = false;
#pragma unroll
            for (int s4 = 0; s4 < NPL; ++s4) {
                const int c = lane + 32 * s4;
                double dd = 0.0;
                if (c < nc) {
                    const long long jj = c0 + c;
                    const double y = ypre[s4];
                    const double xh = best_response(P.S, gv[s4], y, tpre[s4], jj);
                    const double xn = y + P.gamma * (xh - y);
                    xw[jj] = xn;  // every panel writes the same value
                    dd = xn - y;
                }
                if (c < Bpad) dv[c] = dd;
                // the slot's next user accumulates into the other half: clear ALL Bmax entries
                // (that user's block may be wider than this one, e.g. after the ragged last block)
                // (replica r is cleared by panel r mod G: every replica by some panel)
                if (!P.deterministic && c < Bmax)
                    for (long long r = p; r < kPanelRep; r += P.G) gnext[r * Bmax + c] = 0.0;
                nz |= dd != 0.0;
            }
            nz = __any_sync(0xffffffffu, nz);
            __syncwarp();
            sp.mark(2);
            sp.mark(3);
            ASY_TRACE(P, md.t, 8);
            const long long r0 = p * R;
            if (hd.parked) tc_fence_after();
            if (nz) {
                if constexpr (BT >= 16) {
#pragma unroll kRoll
                for (int qq = 0; qq < RPL; ++qq) {
                    long long row;
                    double dsum;
                    if (hd.parked) {
                        // the dot warp's lane layout: s8[2 j + t] = this lane's two columns' share of
                        // row 32 qq + 2 (rq + 4 (j ^ par)) + t
                        double s8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                        const uint32_t trow = tquarter + (uint32_t)((hd.parked - 1) * kSlotCols + qq * cols_per_row);
#pragma unroll
                        for (int c32 = 0; c32 < BT; c32 += 32) {
                            constexpr int n8max = BT < 32 ? BT / 8 : 4;
                            uint32_t uu[16 * n8max];
#pragma unroll
                            for (int q8 = 0; q8 < n8max; ++q8) tmem_ld8(trow + 2 * (c32 + 8 * q8), uu + 16 * q8);
                            tmem_wait_ld();
#pragma unroll
                            for (int sub = 0; sub < n8max / 2; ++sub) {
                                const double2 d2 = *reinterpret_cast<const double2*>(dv + c32 + 16 * sub + 2 * co);
#pragma unroll
                                for (int e = 0; e < 8; ++e)
                                    s8[e] = fma(u2d(uu[32 * sub + 2 * e], uu[32 * sub + 2 * e + 1]), d2.x, s8[e]);
#pragma unroll
                                for (int e = 0; e < 8; ++e)
                                    s8[e] = fma(u2d(uu[32 * sub + 16 + 2 * e], uu[32 * sub + 17 + 2 * e]), d2.y, s8[e]);
                            }
                        }
                        // sum over the eight co lanes (transposing butterfly): lane bit 2 pairs the two
                        // row-pair orders (my j = 0, 2 are the partner's j = 1, 3), bits 3 and 4 split
                        // the remaining four rows
                        const double q0 = s8[0] + __shfl_xor_sync(0xffffffffu, s8[2], 4);
                        const double q1 = s8[1] + __shfl_xor_sync(0xffffffffu, s8[3], 4);
                        const double q2 = s8[4] + __shfl_xor_sync(0xffffffffu, s8[6], 4);
                        const double q3 = s8[5] + __shfl_xor_sync(0xffffffffu, s8[7], 4);
                        const bool up3 = (lane & 8) != 0, up4 = (lane & 16) != 0;
                        const double r0s = (up3 ? q2 : q0) + __shfl_xor_sync(0xffffffffu, up3 ? q0 : q2, 8);
                        const double r1s = (up3 ? q3 : q1) + __shfl_xor_sync(0xffffffffu, up3 ? q1 : q3, 8);
                        dsum = (up4 ? r1s : r0s) + __shfl_xor_sync(0xffffffffu, up4 ? r0s : r1s, 16);
                        row = r0 + 32 * qq + 2 * (rq + 4 * (co & 1) + (up3 ? 8 : 0)) + (up4 ? 1 : 0);
                    } else {
                        double acc4[4] = {0.0, 0.0, 0.0, 0.0};
                        row = r0 + lane + 32 * qq;
                        if (row < P.m) {
                            // re-read the panel row from global memory (L2, usually)
                            const double* a = P.A + c0 * P.lda + row;
#pragma unroll 1
                            for (int c8 = 0; c8 < nc; c8 += 8) {
                                double av[8];
#pragma unroll
                                for (int i = 0; i < 8; ++i) av[i] = (c8 + i) < nc ? __ldg(a + (c8 + i) * P.lda) : 0.0;
#pragma unroll
                                for (int i = 0; i < 8; ++i) acc4[i & 3] = fma(av[i], dv[c8 + i], acc4[i & 3]);
                            }
                        }
                        dsum = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
                    }
#ifdef ASY_DIAG_NO_RED
                    if (row < P.m && dsum == 12345.0) P.r[row] = dsum;
#else
                    if (row < P.m && dsum != 0.0) atomicAdd(&P.r[row], dsum);
#endif
                }
                } else {
#pragma unroll kRoll
                for (int qq = 0; qq < RPL; ++qq) {
                    double acc4[4] = {0.0, 0.0, 0.0, 0.0};
                    const long long row = r0 + lane + 32 * qq;
                    if (hd.parked) {
                        const uint32_t trow = tquarter + (uint32_t)((hd.parked - 1) * kSlotCols + qq * cols_per_row);
#pragma unroll
                        for (int c32 = 0; c32 < BT; c32 += 32) {
                            constexpr int n8max = BT < 32 ? BT / 8 : 4;
                            uint32_t uu[16 * n8max];
#pragma unroll
                            for (int s8 = 0; s8 < n8max; ++s8) tmem_ld8(trow + 2 * (c32 + 8 * s8), uu + 16 * s8);
                            tmem_wait_ld();
#pragma unroll
                            for (int i = 0; i < 8 * n8max; i += 2) {
                                const double2 d2 = *reinterpret_cast<const double2*>(dv + c32 + i);
                                acc4[i & 3] = fma(u2d(uu[2 * i], uu[2 * i + 1]), d2.x, acc4[i & 3]);
                                acc4[(i + 1) & 3] = fma(u2d(uu[2 * i + 2], uu[2 * i + 3]), d2.y, acc4[(i + 1) & 3]);
                            }
                        }
                    } else if (row < P.m) {
                        // re-read the panel row from global memory (L2, usually)
                        const double* a = P.A + c0 * P.lda + row;
#pragma unroll 1
                        for (int c8 = 0; c8 < nc; c8 += 8) {
                            double av[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) av[i] = (c8 + i) < nc ? __ldg(a + (c8 + i) * P.lda) : 0.0;
#pragma unroll
                            for (int i = 0; i < 8; ++i) acc4[i & 3] = fma(av[i], dv[c8 + i], acc4[i & 3]);
                        }
                    }
                    const double dsum = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
#ifdef ASY_DIAG_NO_RED
                    if (row < P.m && dsum == 12345.0) P.r[row] = dsum;
#else
                    if (row < P.m && dsum != 0.0) atomicAdd(&P.r[row], dsum);
#endif
                }
                }
            }
            ASY_TRACE(P, md.t, 9);
            sp.mark(4);
            if (hd.parked) {
                // TMEM slot free.  The loads completed (wait::ld), so a plain store is enough; a
                // release store would also wait for this panel's red.adds to reach L2.
                tc_fence_before();
                __syncwarp();
                ++tm_fin;
                if (lane == 0) st_volatile_cta_u32(&tm_done[ax], tm_fin);
            }
            __syncwarp();
            ASY_TRACE(P, md.t, 7);
            pend_slot = slot;
            pend_b = b;
            pend_k = k;
            sp.mark(5);
        }
        complete();
        sp.flush(P.prof ? P.prof + ((size_t)blockIdx.x * 16 + warp) * 8 : nullptr, lane);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kProducerWarp) tmem_dealloc_512(tmem_base);
}

}  // namespace asy
