// dense_slabt.cuh -- row-slab asynchronous block-update kernel with the tile parked in TMEM.
//
// Same method as dense_slab.cuh (Algorithm 1 [PAPER.md:246-260]; one persistent CTA per
// SM owns rows [row0, row0 + rows) of A, r and b / y; every block update is a grid-wide
// all-reduce of per-slab partials; bounded delay D1 [PAPER.md:224] and own-block
// freshness D4 [PAPER.md:233] enforced per CTA), organised so that HBM streams while
// the all-reduces are in flight:
//
//   * the slab is cut into 32-row groups g.  Dot warp d and axpy warp d share one TMEM lane
//     quarter (warp id mod 4; lane = row) and own the groups g = d + 4 i of the full rounds
//     for the whole launch; the groups of the last, partial round rotate over the warps
//     from one block update to the next (balanced load), a per-group progress counter
//     ordering their updates;
//   * a block's columns are processed as NSPLIT = BMAX / 32 "sub-sequences" of CS = 32
//     columns: each has its own all-reduce, so the all-reduce of columns [0, 32) overlaps
//     the loads and dot of the later columns, and a dot warp can start sub-sequence (k+1, h)
//     as soon as the all-reduce of (k, h) (or an earlier one: spare park slots) has
//     freed its park slots.  The gradient of all sub-sequences is taken from ONE residual snapshot
//     (w = phi'(r) is computed once per sequence and kept in registers), and the axpy of
//     the first sub-sequences goes to a pending buffer (delta) that is added to r together
//     with the last one -- every residual row always holds whole block updates (reading
//     R8 of DESIGN.md is unchanged);
//   * slabs are whole 32-row groups (CTAs own ngt / grid or one more), so every unit is one
//     2-D TMA box of 32 rows x 16 columns (4 KB); lanes 0-7 of warp 1 issue the four dot
//     warps' unit streams (two lanes per stream) in lockstep into per-warp rings of nsw stages.  Units are taken
//     column block by column block across a warp's groups, so one butterfly reduction
//     covers all its rows;
//   * in the same pass over shared memory each unit is parked in its group's park slot
//     (TMEM, tcgen05.st 32x32b; shared-memory hold slots for what does not fit in the
//     256 KB of TMEM) and its stage is refilled immediately;
//   * the axpy warp applies r_g += A[g, cols] dx from the park slot (tcgen05.ld / lds) and
//     frees it.
// Warp 0 only evaluates the schedule (metadata ring, ready flags).  A park slot is waited
// for before the dot pass of a sub-sequence; the ring holds one whole sequence per warp,
// so the slot was used by the previous sequence's same sub-sequence, whose dx only needs
// partials every CTA has already published: no deadlock.
// delay == 0: sequential and bit-reproducible, as in dense_slab.cuh.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "dense_async.cuh"
#include "dense_slab.cuh"

namespace asy {

constexpr int kSlabTMaxStages = 64;  // 4 dot warps x nsw
#ifndef ASY_SLABT_UC
#define ASY_SLABT_UC 32
#endif
constexpr int kSlabTUnitCols = ASY_SLABT_UC;  // columns per unit stage: a 32 x 32 box halves the per-unit
                                              // mbarrier / issue overhead of 32 x 16 boxes
constexpr int kSlabTMaxG = 4;        // row groups per warp per sequence (slabs <= 512 rows)

template <int BMAX, int LOSS, int CS_ = 32>
__global__ void __launch_bounds__(kSlabThreads, 1)
    dense_slabt_kernel(const __grid_constant__ CUtensorMap tmap, const SlabParams P) {
    constexpr int CS = CS_;                    // columns of a sub-sequence (32, or 64 for blocks of 33-64)
    constexpr int NSPLIT = BMAX / CS;          // sub-sequences (all-reduces) per block update
    constexpr int SQ = 256 / CS;               // TMEM park slots per lane quarter (2*CS b32 columns)
    constexpr int UC = kSlabTUnitCols < CS ? kSlabTUnitCols : CS;  // columns of a unit (one TMA box / mbarrier)
    constexpr int NH = UC / 16;                // 16-column halves of a unit
    constexpr int UNIT = 32 * UC;              // doubles per unit stage (4 or 8 KB)
    constexpr int HSLOT = 32 * CS;             // doubles per smem hold slot
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int nsw = P.nst / kSlabDot;
    const int64_t RsP = (P.Rs + 1) & ~(int64_t)1;
    double* dstage = reinterpret_cast<double*>(smem_raw);            // nst * UNIT
    double* hold = dstage + (size_t)P.nst * UNIT;                     // nsa * HSLOT
    double* rs = hold + (size_t)P.nsa * HSLOT;                        // Rs   residual slab
    double* auxs = rs + RsP;                                          // Rs   b / y slab
    double* delta = auxs + RsP;                                       // Rs   pending sub-sequence axpy
    double* wscr = delta + RsP;                                       // kSlabDot * kSlabTMaxG * 32: w = phi'(r) per dot warp
    double* pring = wscr + kSlabDot * kSlabTMaxG * 32;                // NP * kSlabDot * CS
    double* dxring = pring + kSlabNP * kSlabDot * CS;                 // NDX * CS
    SeqMeta* meta = reinterpret_cast<SeqMeta*>(dxring + kSlabNDX * CS);  // NM
    long long* meta_k = reinterpret_cast<long long*>(meta + kSlabNM);    // NM ready flags
    uint64_t* bars = reinterpret_cast<uint64_t*>(meta_k + kSlabNM);
    uint64_t* dfull = bars;                       // nst
    uint64_t* dempty = dfull + kSlabTMaxStages;   // nst
    uint64_t* pfull = dempty + kSlabTMaxStages;   // NP
    uint64_t* pempty = pfull + kSlabNP;           // NP
    uint64_t* dxfull = pempty + kSlabNP;          // NDX
    uint64_t* dxempty = dxfull + kSlabNDX;        // NDX
    uint64_t* arrived = dxempty + kSlabNDX;       // NDX: all CTAs' partials of the slot's sub-sequence
    unsigned long long* progress = reinterpret_cast<unsigned long long*>(arrived + kSlabNDX);  // kSlabAx
    unsigned long long* xprog = progress + kSlabAx;   // kSlabDot: sequences applied to extra group e
    unsigned* parked_done = reinterpret_cast<unsigned*>(xprog + kSlabDot);                     // kSlabDot
    uint32_t* tmem_base_s = parked_done + kSlabDot;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // slabs are whole 32-row groups: CTA s owns groups [gs, gs + ng), ng = base or base + 1; only
    // the matrix's last group can be short (the TMA zero-fills its rows >= m)
    const int64_t ngt = (P.m + 31) / 32, gbase = ngt / gridDim.x, gextra = ngt % gridDim.x;
    const int nrg = (int)(gbase + ((int64_t)blockIdx.x < gextra ? 1 : 0));         // my row groups
    const int64_t row0 = 32 * ((int64_t)blockIdx.x * gbase + min((int64_t)blockIdx.x, gextra));
    const int rows = (int)max((int64_t)0, min((int64_t)32 * nrg, P.m - row0));     // this CTA's slab rows
    const int64_t K = P.K, N = P.nblk;
    const int B = (int)P.B;
    // Row groups of warp d in sequence k: the base groups d + 4 i (i < nb, fixed for the launch)
    // and at most one of the slab's last, partial round ("extra" groups 4 nb + e, e < E), which
    // goes to warp (e + k) mod 4 (rotate) or warp e.  A rotating group's rows are updated by a
    // different axpy warp in each sequence: xprog[e] orders those updates and guards their reads.
    const int nb = nrg / kSlabDot, E = nrg % kSlabDot;
    auto extra_of = [&](int d, int64_t k) {  // extra group index e of warp d in sequence k, or -1
        const int e = P.rotate ? ((d - (int)(k & 3)) & 3) : d;
        return e < E ? e : -1;
    };
    auto cnt_of = [&](int d, int64_t k) { return nb + (extra_of(d, k) >= 0 ? 1 : 0); };
    auto grp_of = [&](int d, int64_t k, int i) { return i < nb ? d + kSlabDot * i : kSlabDot * nb + extra_of(d, k); };

    // ---- init
    for (int64_t i = threadIdx.x; i < (int64_t)P.nst * UNIT + (int64_t)P.nsa * HSLOT; i += blockDim.x) dstage[i] = 0.0;
    for (int i = threadIdx.x; i < kSlabNP * kSlabDot * CS + kSlabNDX * CS; i += blockDim.x) pring[i] = 0.0;
    for (int i = threadIdx.x; i < P.Rs; i += blockDim.x) {
        rs[i] = i < rows ? P.r[row0 + i] : 0.0;
        auxs[i] = i < rows ? P.aux[row0 + i] : 0.0;
        delta[i] = 0.0;
    }
    for (int i = threadIdx.x; i < kSlabNM; i += blockDim.x) meta_k[i] = -1;
    if (warp == 0) tmem_alloc_512(tmem_base_s);
    if (threadIdx.x == 0) {
        for (int s = 0; s < P.nst; ++s) {
            mbar_init(&dfull[s], 1);
            mbar_init(&dempty[s], 1);
        }
        for (int s = 0; s < kSlabNP; ++s) {
            mbar_init(&pfull[s], kSlabDot);
            mbar_init(&pempty[s], 1);
        }
        for (int s = 0; s < kSlabNDX; ++s) {
            mbar_init(&dxfull[s], 1);
            mbar_init(&dxempty[s], kSlabAx);
            mbar_init(&arrived[s], 1);
        }
        for (int a = 0; a < kSlabAx; ++a) progress[a] = 0ull;
        for (int e = 0; e < kSlabDot; ++e) xprog[e] = 0ull;
        for (int d = 0; d < kSlabDot; ++d) parked_done[d] = 0u;
        mbar_fence_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_base_s;
    // zero the TMEM (park slots are written only over the columns of the block's column
    // blocks; the axpy reads whole slots, so the rest must hold finite values)
    if (warp >= kSlabDot0 && warp < kSlabAx0) {
        const uint32_t tq = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
        double z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c = 0; c < 512; c += 16) tmem_st8(tq + (uint32_t)c, z);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    SlabProf sp;
    sp.start();
    if (warp == 0) {
        // ---------------------------------------------------------------- schedule (S.1) + watcher
        // Lane 0 alternates two non-blocking steps: (1) walk the schedule into the metadata
        // ring, up to kSlabNM sequences ahead of the slowest axpy warp; (2) poll the arrival
        // counter of the oldest sub-sequence not yet complete and, once all CTAs arrived,
        // signal its sequence warp (mbarrier arrived[s mod 6]).  One poller per CTA: hundreds
        // of warps polling the counters slow every all-reduce down (measured).
        if (lane == 0) {
            SlabSchedule sch;
            sch.init(N);
            const int64_t total = K * NSPLIT;
            const int64_t S = P.slots;
            int lgS = 0;
            while (((int64_t)1 << lgS) < S) ++lgS;
            const unsigned grid = gridDim.x;
            int64_t ks = 0, sw = 0;
            RingPos wp;
            wp.init(kSlabNDX);
            unsigned ns = 32;
            while (ks < K || sw < total) {
                bool moved = false;
                if (ks < K) {
                    bool room = true;
                    if (ks >= kSlabNM)
                        for (int a = 0; a < kSlabAx; ++a)
                            room = room && ld_acquire_cta_u64(&progress[a]) >= (unsigned long long)(ks - kSlabNM + 1);
                    if (room) {
                        meta[ks & (kSlabNM - 1)] = sch.next(P, ks);
                        asm volatile("st.release.cta.shared.b64 [%0], %1;" ::"r"(smem_u32(&meta_k[ks & (kSlabNM - 1)])),
                                     "l"((long long)ks)
                                     : "memory");
                        ++ks;
                        moved = true;
                    }
                }
                while (sw < total &&
                       ld_relaxed_gpu_u32(&P.arrive[(sw & (S - 1)) * kArrivePad]) >= (unsigned)((sw >> lgS) + 1) * grid) {
                    mbar_arrive(&arrived[wp.i]);
                    wp.next();
                    ++sw;
                    moved = true;
                }
                if (moved) {
                    ns = 32;
                } else {
                    __nanosleep(ns);
                    if (ns < 128) ns <<= 1;
                }
            }
        }
        sp.mark(0);
    } else if (warp == 1) {
        // ---------------------------------------------------------------- loads (all four dot rings)
        // Dot warp d's unit stream: for k, h < NSPLIT, 16-column block cb, i < cnt_d: rows of
        // group d + 4 i, columns [b B + h CS + 16 cb, +16).  The issuing lanes run in lockstep
        // and issue in the same instruction whenever their ring has a free stage (a thread
        // sustains only ~1 bulk copy per ~450 ns, tools/mb_tma.cu), and no ring waits for
        // another (a dot warp waiting for a park slot holds only its own stages).
        const int W = B < UC ? B : UC;  // unit columns loaded
        const uint32_t box_bytes = 32u * (uint32_t)W * 8u;
        const uint64_t pol = policy_evict_first();
        // lanes (d, e), d = lane & 3, e = lane >> 2 < NL: ring d's units u = e (mod NL) go to
        // stage u mod nsw (NL = 2 when nsw is even: eight issuing threads per SM)
        const int NL = (nsw & 1) ? 1 : 2;
        const int d = lane & (kSlabDot - 1), e = lane >> 2;
        int ist = e, first = 1, ih = 0, icb = 0, ii = 0;
        uint32_t iph = 0;
        int64_t ik = e < NL ? 0 : K, icol0 = 0, icached = -1;
        int cnt = 0;
        auto skip = [&]() {  // to the next sequence in which warp d has groups
            while (ik < K && (cnt = cnt_of(d, ik)) == 0) ++ik;
        };
        auto adv = [&]() {  // next unit of ring d
            if (++ii == cnt) {
                ii = 0;
                const int bh = min(CS, B - ih * CS);
                if (++icb == (bh <= 0 ? 0 : (bh + UC - 1) / UC)) {
                    icb = 0;
                    if (++ih == NSPLIT) {
                        ih = 0;
                        ++ik;
                        skip();
                    }
                }
            }
        };
        skip();
        if (ik < K && e == 1) adv();
        for (;;) {
            const bool live = ik < K;
            if (!__any_sync(0xffffffffu, live)) break;
            bool ok = false;
            const int st = d * nsw + ist;
            if (live) {
                ok = first || mbar_test(&dempty[st], iph ^ 1u);
                if (ok && icached != ik) {
                    long long v;
                    asm volatile("ld.acquire.cta.shared.b64 %0, [%1];"
                                 : "=l"(v)
                                 : "r"(smem_u32(&meta_k[ik & (kSlabNM - 1)]))
                                 : "memory");
                    ok = v == ik;
                    if (ok) {
                        icol0 = (int64_t)meta[ik & (kSlabNM - 1)].b * P.B;
                        icached = ik;
                    }
                }
            }
            if (ok) {
                const int g = grp_of(d, ik, ii);
                mbar_arrive_expect_tx(&dfull[st], box_bytes);
                slab_tma_2d(dstage + (size_t)st * UNIT, &tmap, (int)(row0 + 32 * g), (int)(icol0 + ih * CS + icb * UC),
                            &dfull[st], pol);
                ist += NL;
                if (ist >= nsw) { ist -= nsw; iph ^= 1u; first = 0; }
                adv();
                if (NL == 2 && ik < K) adv();
            }
            if (!__any_sync(0xffffffffu, ok)) __nanosleep(32);
        }
        sp.mark(0);
    } else if (warp < kSlabAx0) {
        // ---------------------------------------------------------------- dot warps
        const int d = warp - kSlabDot0;
        const uint32_t tq = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
        const int np = P.npark[d];
        double* myhold = hold + (size_t)P.hoff[d] * HSLOT;
        uint64_t* myfull = dfull + d * nsw;
        uint64_t* myempty = dempty + d * nsw;
        const double* mystage = dstage + (size_t)d * nsw * UNIT;
        // column blocks of sub-sequence h (blocks narrower than BMAX skip the empty ones)
        auto ncb_of = [&](int h) {  // units of sub-sequence h
            const int bh = min(CS, B - h * CS);
            return bh <= 0 ? 0 : (bh + UC - 1) / UC;
        };
        RingPos pp;
        pp.init(kSlabNP);
        RingPos cr;         // consumed units: stage, phase
        cr.init(nsw);
        unsigned used = 0;  // park slots taken
        int pslot = 0;      // used mod np
        long long dmax_local = 0;
        // Lane layout of a 32 x 16 unit (see the header): lane (co = lane >> 2, rq = lane & 3)
        // owns columns 2 co, 2 co + 1 and the row pairs rq + 4 (j ^ (co & 1)), j < 4, read as
        // double2 (8 conflict-free 16-byte loads per unit); the sum over rows is then in-lane
        // except for the four rq lanes (two shuffles per 16-column block).
        const int rq = lane & 3, co = lane >> 2;
        const int lbase = 64 * co + 2 * rq;                       // doubles: column 2 co, row 2 rq
        const int o0 = 8 * (co & 1), o1 = 8 - o0;                 // row-pair offsets of j = 0, 1 (j = 2, 3: + 16)
        double* mywscr = wscr + d * kSlabTMaxG * 32;
        for (int64_t k = 0; k < K; ++k) {
            const int cnt = cnt_of(d, k);  // my row groups in sequence k
            const int ex = extra_of(d, k);
            if (cnt > 0) {
                // D1 / D4 guards: axpy(k - delay - 1) and axpy(kprev) applied to my rows.  Every lane
                // polls (broadcast shared-memory loads): no lane-0 branch, no warp barrier
                for (;;) {
                    long long v;
                    asm volatile("ld.acquire.cta.shared.b64 %0, [%1];"
                                 : "=l"(v)
                                 : "r"(smem_u32(&meta_k[k & (kSlabNM - 1)]))
                                 : "memory");
                    if (v == k) break;
                    __nanosleep(32);
                }
                sp.mark(4);
                const int64_t need = meta[k & (kSlabNM - 1)].need;
                // observed delay: the rows about to be read lack exactly sequences progress..k-1
                unsigned long long have = nb > 0 ? ld_acquire_cta_u64(&progress[d]) : (unsigned long long)k;
                if (ex >= 0) {
                    const unsigned long long hx = ld_acquire_cta_u64(&xprog[ex]);
                    if (hx < have) have = hx;
                }
                while ((long long)have < need) {
                    __nanosleep(20);
                    have = nb > 0 ? ld_acquire_cta_u64(&progress[d]) : (unsigned long long)k;
                    if (ex >= 0) {
                        const unsigned long long hx = ld_acquire_cta_u64(&xprog[ex]);
                        if (hx < have) have = hx;
                    }
                }
                {
                    const long long miss = k - (long long)have;
                    if (miss > dmax_local) dmax_local = miss;
                }
                sp.mark(1);
                // one residual snapshot for the whole block update (lane = row here; the dot pass
                // reads it back per row pair)
                __syncwarp();
                for (int i = 0; i < cnt; ++i) {
                    const int srow = 32 * grp_of(d, k, i) + lane;
                    mywscr[i * 32 + lane] = srow < rows ? loss_prime_t<LOSS>(P.S, rs[srow], auxs[srow]) : 0.0;
                }
                __syncwarp();
            }
#pragma unroll 1
            for (int h = 0; h < NSPLIT; ++h) {
                const int ncb = cnt > 0 ? ncb_of(h) : 0;
                // partial ring slot of sub-sequence s = k * NSPLIT + h
                if (k * NSPLIT + h >= kSlabNP) mbar_wait(&pempty[pp.i], pp.ph ^ 1u);
                double* pdst = pring + (size_t)(pp.i * kSlabDot + d) * CS;
                if (ncb > 0) {
                    // park slots used..used+cnt-1: free once the axpy consumed the slots parked np ago
                    if (used + (unsigned)cnt > (unsigned)np) {
                        const unsigned want = used + (unsigned)cnt - (unsigned)np;
                        while (ld_acquire_cta_u32(&parked_done[d]) < want) __nanosleep(20);
                    }
                    tc_fence_after();
                    sp.mark(5);
                    const int bhh = min(CS, B - h * CS);  // columns of this sub-sequence
#pragma unroll 1
                    for (int cb = 0; cb < ncb; ++cb) {
                        // acc[hf][0..3]: columns 2 co (x, y rows), 2 co + 1 of 16-column half hf of the unit
                        double acc[NH][4];
#pragma unroll
                        for (int hf = 0; hf < NH; ++hf) acc[hf][0] = acc[hf][1] = acc[hf][2] = acc[hf][3] = 0.0;
#pragma unroll 1
                        for (int i = 0; i < cnt; ++i) {
                            const int st = cr.i;
                            sp.mark(3);
                            mbar_wait(&myfull[st], cr.ph);
                            sp.mark(6);
                            const double* wp = mywscr + i * 32 + 2 * rq;
                            double2 wv[4];
                            wv[0] = *reinterpret_cast<const double2*>(wp + o0);
                            wv[1] = *reinterpret_cast<const double2*>(wp + o1);
                            wv[2] = *reinterpret_cast<const double2*>(wp + 16 + o0);
                            wv[3] = *reinterpret_cast<const double2*>(wp + 16 + o1);
                            int ps = pslot + i;
                            if (ps >= np) ps -= np;
#pragma unroll
                            for (int hf = 0; hf < NH; ++hf) {
                                if (hf > 0 && UC * cb + 16 * hf >= bhh) break;  // (no block columns in this half)
                                const double* a = mystage + (size_t)st * UNIT + hf * 16 * 32 + lbase;
                                double v[16];  // v[8 cc + 2 j + t] = A[row 2 (rq + 4 (j ^ par)) + t][column 2 co + cc]
#pragma unroll
                                for (int cc = 0; cc < 2; ++cc) {
                                    const double2 t0 = *reinterpret_cast<const double2*>(a + 32 * cc + o0);
                                    const double2 t1 = *reinterpret_cast<const double2*>(a + 32 * cc + o1);
                                    const double2 t2 = *reinterpret_cast<const double2*>(a + 32 * cc + 16 + o0);
                                    const double2 t3 = *reinterpret_cast<const double2*>(a + 32 * cc + 16 + o1);
                                    v[8 * cc + 0] = t0.x; v[8 * cc + 1] = t0.y;
                                    v[8 * cc + 2] = t1.x; v[8 * cc + 3] = t1.y;
                                    v[8 * cc + 4] = t2.x; v[8 * cc + 5] = t2.y;
                                    v[8 * cc + 6] = t3.x; v[8 * cc + 7] = t3.y;
                                }
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    acc[hf][0] = fma(v[2 * j], wv[j].x, acc[hf][0]);
                                    acc[hf][1] = fma(v[2 * j + 1], wv[j].y, acc[hf][1]);
                                    acc[hf][2] = fma(v[8 + 2 * j], wv[j].x, acc[hf][2]);
                                    acc[hf][3] = fma(v[8 + 2 * j + 1], wv[j].y, acc[hf][3]);
                                }
                                const int cb16 = NH * cb + hf;  // 16-column block of the sub-sequence
                                if (ps < SQ) {
                                    const uint32_t t = tq + (uint32_t)(ps * 2 * CS + 2 * 16 * cb16);
                                    tmem_st8(t, v);
                                    tmem_st8(t + 16, v + 8);
                                } else {
                                    double* hp = myhold + (size_t)(ps - SQ) * HSLOT + cb16 * 16 * 32 + lane;
#pragma unroll
                                    for (int c = 0; c < 16; ++c) hp[c * 32] = v[c];
                                }
                            }
                            sp.mark(2);
                            __syncwarp();       // every lane's reads of the stage are done
                            if (lane == 0) mbar_arrive(&myempty[st]);
                            cr.next();
                        }
                        sp.mark(3);
                        // columns 2 co, 2 co + 1 summed over the four rq lanes: lanes with rq & 1 == c
                        // end with column 2 co + c
#pragma unroll
                        for (int hf = 0; hf < NH; ++hf) {
                            const double s0 = acc[hf][0] + acc[hf][1], s1 = acc[hf][2] + acc[hf][3];
                            const bool up = (lane & 1) != 0;
                            double cs_ = (up ? s1 : s0) + __shfl_xor_sync(0xffffffffu, up ? s0 : s1, 1);
                            cs_ += __shfl_xor_sync(0xffffffffu, cs_, 2);
                            if (rq < 2 && (NH * cb + hf) * 16 < CS) pdst[(NH * cb + hf) * 16 + 2 * co + rq] = cs_;
                        }
                        sp.mark(7);
                    }
                    used += (unsigned)cnt;
                    pslot += cnt;
                    if (pslot >= np) pslot -= np;
                    tmem_wait_st();
                    tc_fence_before();
                    sp.mark(0);
                } else {
                    // no rows (or no columns in this sub-sequence): a zero partial
                    for (int c = lane; c < CS; c += 32) pdst[c] = 0.0;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfull[pp.i]);
                pp.next();
                sp.mark(4);
            }
        }
        if (lane == 0 && P.dobs) atomicMax(P.dobs, (unsigned)dmax_local);
    } else if (warp < kSlabSeq0) {
        // ---------------------------------------------------------------- axpy warps
        const int a = warp - kSlabAx0;  // same TMEM lane quarter and rows as dot warp a
        const uint32_t tq = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
        const int np = P.npark[a];
        const double* myhold = hold + (size_t)P.hoff[a] * HSLOT;
        RingPos xp;
        xp.init(kSlabNDX);
        unsigned fin = 0;
        int pslot = 0;
        const int rq = lane & 3, co = lane >> 2;  // the dot warps' lane layout
        for (int64_t s = 0; s < K * NSPLIT; ++s) {
            const int64_t k = s / NSPLIT;
            const int h = (int)(s - k * NSPLIT);
            const int bh = min(CS, B - h * CS);
            const int cnt = cnt_of(a, k), ex = extra_of(a, k);
            mbar_wait(&dxfull[xp.i], xp.ph);
            sp.mark(1);
            // a rotating group: the previous sequence's update of its rows (another warp) first
            if (h == 0 && ex >= 0)
                while (ld_acquire_cta_u64(&xprog[ex]) < (unsigned long long)k) __nanosleep(20);
            const double* dxv = dxring + xp.i * CS;
            if (bh > 0) {
                for (int i = 0; i < cnt; ++i) {
                    double s8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // s8[2 j + t]: row 2 (rq + 4 (j ^ par)) + t
                    int ps = pslot + i;
                    if (ps >= np) ps -= np;
                    if (ps < SQ) {
                        tc_fence_after();
                        const uint32_t t = tq + (uint32_t)(ps * 2 * CS);
#pragma unroll
                        for (int c32 = 0; c32 < CS; c32 += 16) {
                            uint32_t uu[32];
#pragma unroll
                            for (int q8 = 0; q8 < 2; ++q8) tmem_ld8(t + (uint32_t)(2 * (c32 + 8 * q8)), uu + 16 * q8);
                            tmem_wait_ld();
                            const double2 d2 = *reinterpret_cast<const double2*>(dxv + c32 + 2 * co);
#pragma unroll
                            for (int e = 0; e < 8; ++e) s8[e] = fma(u2d(uu[2 * e], uu[2 * e + 1]), d2.x, s8[e]);
#pragma unroll
                            for (int e = 0; e < 8; ++e) s8[e] = fma(u2d(uu[16 + 2 * e], uu[17 + 2 * e]), d2.y, s8[e]);
                        }
                        tc_fence_before();
                    } else {
                        const double* t = myhold + (size_t)(ps - SQ) * HSLOT + lane;
#pragma unroll 1
                        for (int c32 = 0; c32 < CS; c32 += 16) {
                            const double2 d2 = *reinterpret_cast<const double2*>(dxv + c32 + 2 * co);
#pragma unroll
                            for (int e = 0; e < 8; ++e) s8[e] = fma(t[(c32 + e) * 32], d2.x, s8[e]);
#pragma unroll
                            for (int e = 0; e < 8; ++e) s8[e] = fma(t[(c32 + 8 + e) * 32], d2.y, s8[e]);
                        }
                    }
                    // the park slot is free as soon as every lane holds its elements' products (the
                    // row sums below and the residual update do not read it)
                    __syncwarp();
                    ++fin;
                    if (lane == 0) st_release_cta_u32(&parked_done[a], fin);
                    // sum over the eight co lanes (transposing butterfly): lane bit 2 pairs the two
                    // row-pair orders (my j = 0, 2 are the partner's j = 1, 3), bits 3 and 4 split the
                    // remaining four rows; the lane ends with the total of row
                    // 2 (rq + 4 par + 8 b3) + b4
                    const double q0 = s8[0] + __shfl_xor_sync(0xffffffffu, s8[2], 4);
                    const double q1 = s8[1] + __shfl_xor_sync(0xffffffffu, s8[3], 4);
                    const double q2 = s8[4] + __shfl_xor_sync(0xffffffffu, s8[6], 4);
                    const double q3 = s8[5] + __shfl_xor_sync(0xffffffffu, s8[7], 4);
                    const bool up3 = (lane & 8) != 0, up4 = (lane & 16) != 0;
                    const double r0 = (up3 ? q2 : q0) + __shfl_xor_sync(0xffffffffu, up3 ? q0 : q2, 8);
                    const double r1 = (up3 ? q3 : q1) + __shfl_xor_sync(0xffffffffu, up3 ? q1 : q3, 8);
                    const double part = (up4 ? r1 : r0) + __shfl_xor_sync(0xffffffffu, up4 ? r0 : r1, 16);
                    const int srow = 32 * grp_of(a, k, i) + 2 * (rq + 4 * (co & 1) + (up3 ? 8 : 0)) + (up4 ? 1 : 0);
                    if (srow < rows) {
                        if (NSPLIT == 1) rs[srow] += part;
                        else if (h == 0) delta[srow] = part;
                        else if (h < NSPLIT - 1) delta[srow] += part;
                        else rs[srow] += delta[srow] + part;  // the whole block update at once
                    }
                }
                pslot += cnt;
                if (pslot >= np) pslot -= np;
            } else if (h == NSPLIT - 1) {
                // (a block narrower than the split: its update is complete in delta)
                for (int i = 0; i < cnt; ++i) {
                    const int srow = 32 * grp_of(a, k, i) + lane;
                    if (srow < rows) rs[srow] += delta[srow];
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&dxempty[xp.i]);
                if (h == NSPLIT - 1) {
                    if (ex >= 0) st_release_cta_u64(&xprog[ex], (unsigned long long)(k + 1));
                    st_release_cta_u64(&progress[a], (unsigned long long)(k + 1));
                }
            }
            xp.next();
            sp.mark(4);
        }
    } else {
        slab_sequence_warp<BMAX, NSPLIT>(P, warp - kSlabSeq0, lane, pring, dxring, meta, pfull, pempty, dxfull,
                                          dxempty, sp, arrived, meta_k);
    }
    sp.flush(P.prof ? P.prof + ((size_t)blockIdx.x * kSlabWarps + warp) * 8 : nullptr, lane);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc_512(tmem_base);
    for (int i = threadIdx.x; i < rows; i += blockDim.x) P.r[row0 + i] = rs[i];
}

}  // namespace asy
