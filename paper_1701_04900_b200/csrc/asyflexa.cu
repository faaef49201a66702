// asyflexa.cu -- host runtime behind the C ABI of include/asyflexa.h.
//
// Owns device memory, validates the problem statement (problem (1)
// [PAPER.md:58-68]), launches the kernels of dense_async.cuh,
// sparse_async.cuh and sync_kernels.cuh on the handle's stream, and times the
// update kernels with CUDA events on that stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "../../include/asyflexa.h"
#include "common.cuh"
#include "dense_async.cuh"
#include "dense_slab.cuh"
#include "dense_slabt.cuh"
#include "sparse_async.cuh"
#include "sync_kernels.cuh"

using namespace asy;

static std::string g_create_error;

// Developer knobs (traces, segment profiles, geometry sweeps) exist only in a debug build
// (-DASY_DEBUG_KNOBS: `python -m paper_1701_04900_b200.build --variant debug ASY_DEBUG_KNOBS`,
// loaded with ASY_LIB_VARIANT=debug).  The product library reads no environment variable:
// kernel choice and geometry overrides come through asy_solve_params.tuning.
static const char* dbg_env(const char* name) {
#ifdef ASY_DEBUG_KNOBS
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

static const asy_tuning kNoTuning{};
static const asy_tuning& tuning_of(const asy_solve_params* sp) { return sp->tuning ? *sp->tuning : kNoTuning; }

struct Dev {
    void* p = nullptr;
    size_t bytes = 0;
    bool own = false;
};

struct asy_handle {
    int device = 0;
    int sms = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

    // problem
    bool has_problem = false;
    int kind = 0, loss = 0, reg = 0;
    int64_t m = 0, n = 0, lda = 0, nnz = 0, B = 1, nblk = 0;
    Scalars S{};
    Dev A, colptr, rowidx, vals;          // borrowed or owned
    Dev rowptr, csr_col, csr_val;         // CSR transpose (owned)
    Dev b, tau, lo, hi;                   // owned copies
    // state
    Dev x, xalt, r, dx, w, mf, mer, rs, xs;  // xalt: 2nd half of the async x double buffer; rs/xs: scratch
    Dev part;                             // GEMV-N partial sums
    int64_t gemv_chunks = 1, gemv_cpc = 1;
    Dev red_part, red_out;                // reduction buffers
    // async state
    Dev counter, gacc, dpart, arrive, consumed, done, ver, wcnt;
    Dev dobs;                             // observed-delay statistic (u32)
    int64_t slots = 0;
    int64_t epochs = 0;                   // sweeps since reset (schedule epoch)
    int last_kernel = 0, last_delay = -1; // reported in asy_solve_stats
    int last_dobs = -1;                   // observed delay of the last solve (-1: not measured)

    int fail(int code, const char* fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        return code;
    }
};

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return h->fail(ASY_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),   \
                           __FILE__, __LINE__);                                                   \
    } while (0)
#define CKL()                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = cudaGetLastError();                                                      \
        if (e_ != cudaSuccess)                                                                    \
            return h->fail(ASY_ERR_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                           __FILE__, __LINE__);                                                   \
    } while (0)
#define TRY(expr)                  \
    do {                           \
        int rc_ = (expr);          \
        if (rc_ != ASY_OK) return rc_; \
    } while (0)

static void dev_free(Dev& d) {
    if (d.own && d.p) cudaFree(d.p);
    d = Dev{};
}

static int dev_alloc(asy_handle* h, Dev& d, size_t bytes) {
    if (d.own && d.bytes >= bytes && d.p) return ASY_OK;
    dev_free(d);
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(&d.p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        d = Dev{};
        return h->fail(ASY_ERR_NOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
    d.bytes = bytes;
    d.own = true;
    return ASY_OK;
}

template <typename T>
static T* P_(Dev& d) { return reinterpret_cast<T*>(d.p); }

static int copy_in(asy_handle* h, Dev& d, const void* src, size_t bytes, int mem) {
    TRY(dev_alloc(h, d, bytes));
    CK(cudaMemcpyAsync(d.p, src, bytes, mem == ASY_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                       h->stream));
    return ASY_OK;
}

static inline int grid_for(int64_t n, int threads, int cap) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

static int64_t next_pow2(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

// problem-owned buffers (the handle-lifetime ones -- red_part, red_out, counter -- survive)
static void free_problem(asy_handle* h) {
    Dev* all[] = {&h->A, &h->colptr, &h->rowidx, &h->vals, &h->rowptr, &h->csr_col, &h->csr_val, &h->b,
                  &h->tau, &h->lo, &h->hi, &h->x, &h->xalt, &h->r, &h->dx, &h->w, &h->mf, &h->mer, &h->rs, &h->xs,
                  &h->part, &h->gacc, &h->dpart, &h->arrive, &h->consumed, &h->done,
                  &h->ver, &h->dobs, &h->wcnt};
    for (Dev* d : all) dev_free(*d);
    h->has_problem = false;
}

// Before installing a new problem: forget borrowed arrays, KEEP owned device buffers (dev_alloc
// reuses them when large enough), so re-installing a problem of the same shape -- the e2e path,
// a new right-hand side -- does no cudaFree / cudaMalloc (each of which synchronises the device).
static void release_borrowed(asy_handle* h) {
    Dev* all[] = {&h->A, &h->colptr, &h->rowidx, &h->vals};
    for (Dev* d : all)
        if (!d->own) *d = Dev{};
    h->has_problem = false;
}

static void free_all(asy_handle* h) {
    free_problem(h);
    dev_free(h->red_part);
    dev_free(h->red_out);
    dev_free(h->counter);
}

// --------------------------------------------------------------------------
// device building blocks
// --------------------------------------------------------------------------

// out = A v (+ base per mode), deterministic.  Dense: split partial + combine; CSC: CSR rows.
static int gemvN(asy_handle* h, const double* v, int mode, double* out) {
    if (h->kind == ASY_DENSE_COLMAJOR) {
        dim3 grid((unsigned)((h->m + 255) / 256), (unsigned)h->gemv_chunks);
        dense_gemvN_partial_kernel<<<grid, 256, 0, h->stream>>>(P_<double>(h->A), h->lda, h->m, h->n, v,
                                                                h->gemv_cpc, P_<double>(h->part));
        CKL();
        combine_kernel<<<grid_for(h->m, 256, 4 * h->sms), 256, 0, h->stream>>>(
            P_<double>(h->part), h->gemv_chunks, h->m, mode, P_<double>(h->b), out);
        CKL();
    } else {
        csr_gemvN_kernel<<<grid_for(h->m * 8, 256, 8 * h->sms), 256, 0, h->stream>>>(
            P_<int64_t>(h->rowptr), P_<int32_t>(h->csr_col), P_<double>(h->csr_val), h->m, v, mode,
            P_<double>(h->b), out);
        CKL();
    }
    return ASY_OK;
}

// g = A^T w with the per-coordinate epilogue (Jacobi update or stationarity terms).
static int gemvT(asy_handle* h, const double* w, int mode, double* x, double gamma, double* dx,
                 double* mf, double* mer) {
    if (h->kind == ASY_DENSE_COLMAJOR) {
        dense_gemvT_kernel<<<grid_for(h->n * 32, 256, 16 * h->sms), 256, 0, h->stream>>>(
            P_<double>(h->A), h->lda, h->m, h->n, w, h->S, mode, x, P_<double>(h->tau), gamma, dx, mf, mer);
    } else {
        csc_gemvT_kernel<<<grid_for(h->n * 8, 256, 16 * h->sms), 256, 0, h->stream>>>(
            P_<int64_t>(h->colptr), P_<int32_t>(h->rowidx), P_<double>(h->vals), h->n, w, h->S, mode, x,
            P_<double>(h->tau), gamma, dx, mf, mer);
    }
    CKL();
    return ASY_OK;
}

// out6 (host) = {sum phi(r), sum x^2, sum h(x), #box violations, sum mf^2, max|mf|}
static int reduce_objective(asy_handle* h, const double* r, const double* x, const double* mf, double out6[6]) {
    objective_partial_kernel<<<kRedGrid, kRedThreads, 0, h->stream>>>(h->S, r, P_<double>(h->b), h->m, x, h->n, mf,
                                                                      P_<double>(h->red_part));
    CKL();
    reduce_final_kernel<<<1, 32, 0, h->stream>>>(P_<double>(h->red_part), kRedGrid, 1 << 5, P_<double>(h->red_out));
    CKL();
    CK(cudaMemcpyAsync(out6, h->red_out.p, 6 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return ASY_OK;
}

static double objective_from(const asy_handle* h, const double v[6], double* smooth) {
    const double f = v[0] - 0.5 * h->S.c2 * v[1];
    if (smooth) *smooth = f;
    if (v[3] > 0) return INFINITY;
    return f + h->S.lam * v[2];
}

static int reset_state(asy_handle* h, const double* x0, int x_mem) {
    if (x0) {
        CK(cudaMemcpyAsync(h->x.p, x0, h->n * sizeof(double),
                           x_mem == ASY_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
        TRY(gemvN(h, P_<double>(h->x), h->loss == ASY_LOSS_LS ? COMBINE_FRESH_LS : COMBINE_FRESH_ZERO,
                  P_<double>(h->r)));
    } else {
        // x0 = P_X(0); r = A x0 - b (the GEMV skips the zero columns of x0)
        project_zero_kernel<<<grid_for(h->n, 256, 4 * h->sms), 256, 0, h->stream>>>(h->S, P_<double>(h->x), h->n);
        CKL();
        TRY(gemvN(h, P_<double>(h->x), h->loss == ASY_LOSS_LS ? COMBINE_FRESH_LS : COMBINE_FRESH_ZERO,
                  P_<double>(h->r)));
    }
    h->epochs = 0;
    return ASY_OK;
}

// --------------------------------------------------------------------------
// C ABI
// --------------------------------------------------------------------------
extern "C" {

ASY_API const char* asy_version(void) { return "asyflexa-b200 0.1 (sm_100a)"; }

ASY_API const char* asy_last_error(const asy_handle* h) {
    return h ? h->err.c_str() : g_create_error.c_str();
}

ASY_API void asy_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    philox4x32_10(ctr, key, out);
}

ASY_API int asy_schedule_block(int32_t schedule, uint64_t seed, int64_t nblocks, int64_t k, int64_t* out) {
    if (!out || nblocks < 1 || k < 0 || (schedule != ASY_SCHED_CYCLIC && schedule != ASY_SCHED_RANDOM))
        return ASY_ERR_INVALID;
    *out = schedule_block(schedule, seed, nblocks, k);
    return ASY_OK;
}

ASY_API int asy_schedule_prev(int32_t schedule, uint64_t seed, int64_t nblocks, int64_t k, int64_t* out) {
    if (!out || nblocks < 1 || k < 0 || (schedule != ASY_SCHED_CYCLIC && schedule != ASY_SCHED_RANDOM))
        return ASY_ERR_INVALID;
    *out = schedule_prev(schedule, seed, nblocks, k, schedule_block(schedule, seed, nblocks, k));
    return ASY_OK;
}

ASY_API int asy_create(int device, void* stream, asy_handle** out) {
    if (!out) {
        g_create_error = "asy_create: out is NULL";
        return ASY_ERR_INVALID;
    }
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        g_create_error = std::string("asy_create: no CUDA device: ") + cudaGetErrorString(e);
        return ASY_ERR_CUDA;
    }
    if (device < 0 || device >= ndev) {
        g_create_error = "asy_create: device index out of range";
        return ASY_ERR_INVALID;
    }
    asy_handle* h = new asy_handle();
    h->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        g_create_error = "asy_create: cudaSetDevice failed";
        delete h;
        return ASY_ERR_CUDA;
    }
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    if (prop.major < 10) {
        g_create_error = "asy_create: needs compute capability 10.x (sm_100a)";
        delete h;
        return ASY_ERR_UNSUPPORTED;
    }
    h->sms = prop.multiProcessorCount;
    if (stream) {
        h->stream = reinterpret_cast<cudaStream_t>(stream);
    } else {
        if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
            g_create_error = "asy_create: stream creation failed";
            delete h;
            return ASY_ERR_CUDA;
        }
        h->own_stream = true;
    }
    for (auto& ev : h->ev) cudaEventCreate(&ev);
    if (dev_alloc(h, h->red_part, sizeof(double) * kRedGrid * kRedVals) != ASY_OK ||
        dev_alloc(h, h->red_out, sizeof(double) * 8) != ASY_OK ||
        dev_alloc(h, h->counter, 64) != ASY_OK) {
        g_create_error = h->err;
        free_all(h);
        delete h;
        return ASY_ERR_NOMEM;
    }
    *out = h;
    return ASY_OK;
}

ASY_API int asy_destroy(asy_handle* h) {
    if (!h) return ASY_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    free_all(h);
    for (auto& ev : h->ev)
        if (ev) cudaEventDestroy(ev);
    if (h->own_stream) cudaStreamDestroy(h->stream);
    delete h;
    return ASY_OK;
}

ASY_API int asy_set_problem(asy_handle* h, const asy_problem* p) {
    if (!h) return ASY_ERR_INVALID;
    if (!p) return h->fail(ASY_ERR_INVALID, "asy_set_problem: problem is NULL");
    CK(cudaSetDevice(h->device));
    if (p->m < 1 || p->n < 1) return h->fail(ASY_ERR_INVALID, "m and n must be >= 1");
    if (p->mem != ASY_MEM_HOST && p->mem != ASY_MEM_DEVICE) return h->fail(ASY_ERR_INVALID, "bad mem kind");
    if (p->kind != ASY_DENSE_COLMAJOR && p->kind != ASY_CSC) return h->fail(ASY_ERR_INVALID, "bad matrix kind");
    if (p->loss != ASY_LOSS_LS && p->loss != ASY_LOSS_LOGISTIC) return h->fail(ASY_ERR_INVALID, "bad loss");
    if (p->reg != ASY_REG_L1 && p->reg != ASY_REG_EXP && p->reg != ASY_REG_LOG)
        return h->fail(ASY_ERR_INVALID, "bad regularizer");
    if (p->loss == ASY_LOSS_LS && !(p->loss_scale > 0)) return h->fail(ASY_ERR_INVALID, "loss_scale must be > 0");
    if (!(p->c_nonconvex >= 0) || !(p->lambda >= 0)) return h->fail(ASY_ERR_INVALID, "c and lambda must be >= 0");
    if (p->reg != ASY_REG_L1 && !(p->theta > 0)) return h->fail(ASY_ERR_INVALID, "theta must be > 0");
    if (p->block_size < 1 || p->block_size > 128) return h->fail(ASY_ERR_INVALID, "block_size must be in [1,128]");
    if (!p->b || !p->tau) return h->fail(ASY_ERR_INVALID, "b and tau are required");
    if (!p->lo && !p->hi && !(p->lo_all <= p->hi_all)) return h->fail(ASY_ERR_INVALID, "lo_all > hi_all");
    if ((p->lo == nullptr) != (p->hi == nullptr)) return h->fail(ASY_ERR_INVALID, "lo and hi must both be set or both NULL");
    if (p->kind == ASY_DENSE_COLMAJOR) {
        if (!p->A) return h->fail(ASY_ERR_INVALID, "A is NULL");
        if (p->lda < p->m) return h->fail(ASY_ERR_INVALID, "lda < m");
    } else {
        if (!p->colptr || !p->rowidx || !p->vals) return h->fail(ASY_ERR_INVALID, "CSC arrays are NULL");
        if (p->nnz < 0 || p->nnz >= (int64_t)1 << 31) return h->fail(ASY_ERR_INVALID, "nnz out of range");
    }
    CK(cudaStreamSynchronize(h->stream));
    release_borrowed(h);
    const int cm = p->mem;
    h->kind = p->kind;
    h->loss = p->loss;
    h->reg = p->reg;
    h->m = p->m;
    h->n = p->n;
    h->B = p->block_size;
    h->nblk = (p->n + p->block_size - 1) / p->block_size;

    // ---- matrix
    if (p->kind == ASY_DENSE_COLMAJOR) {
        const bool aligned = (reinterpret_cast<uintptr_t>(p->A) % 16) == 0 && (p->lda % 2) == 0;
        if (cm == ASY_MEM_DEVICE && aligned) {
            dev_free(h->A);  // (an owned copy of a previous problem)
            h->A.p = const_cast<double*>(p->A);
            h->A.own = false;
            h->lda = p->lda;
        } else {
            h->lda = (p->m + 15) / 16 * 16;
            TRY(dev_alloc(h, h->A, sizeof(double) * h->lda * p->n));
            if (h->lda != p->m) CK(cudaMemsetAsync(h->A.p, 0, sizeof(double) * h->lda * p->n, h->stream));
            CK(cudaMemcpy2DAsync(h->A.p, sizeof(double) * h->lda, p->A, sizeof(double) * p->lda,
                                 sizeof(double) * p->m, p->n,
                                 cm == ASY_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
        }
        // GEMV-N split: ~4 waves of 256-row tiles over the SMs
        const int64_t tiles = (h->m + 255) / 256;
        int64_t chunks = std::max<int64_t>(1, (4 * h->sms + tiles - 1) / tiles);
        chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, h->n / 8));
        h->gemv_cpc = (h->n + chunks - 1) / chunks;
        h->gemv_chunks = (h->n + h->gemv_cpc - 1) / h->gemv_cpc;
        TRY(dev_alloc(h, h->part, sizeof(double) * h->gemv_chunks * h->m));
    } else {
        h->nnz = p->nnz;
        if (cm == ASY_MEM_DEVICE) {
            dev_free(h->colptr);
            dev_free(h->rowidx);
            dev_free(h->vals);
            h->colptr.p = const_cast<int64_t*>(p->colptr);
            h->rowidx.p = const_cast<int32_t*>(p->rowidx);
            h->vals.p = const_cast<double*>(p->vals);
        } else {
            TRY(copy_in(h, h->colptr, p->colptr, sizeof(int64_t) * (p->n + 1), cm));
            TRY(copy_in(h, h->rowidx, p->rowidx, sizeof(int32_t) * std::max<int64_t>(1, p->nnz), cm));
            TRY(copy_in(h, h->vals, p->vals, sizeof(double) * std::max<int64_t>(1, p->nnz), cm));
        }
        // check colptr ends
        int64_t ends[2];
        CK(cudaMemcpyAsync(&ends[0], P_<int64_t>(h->colptr), sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(&ends[1], P_<int64_t>(h->colptr) + p->n, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (ends[0] != 0 || ends[1] != p->nnz) {
            free_problem(h);
            return h->fail(ASY_ERR_INVALID, "colptr[0] must be 0 and colptr[n] == nnz");
        }
        // CSR transpose (deterministic: stable radix sort of row keys over column-major order)
        const int64_t nnz = std::max<int64_t>(1, p->nnz);
        Dev colid, perm, keys_out, counts;
        TRY(dev_alloc(h, colid, sizeof(int32_t) * nnz));
        TRY(dev_alloc(h, perm, sizeof(int32_t) * nnz));
        TRY(dev_alloc(h, keys_out, sizeof(int32_t) * nnz));
        TRY(dev_alloc(h, counts, sizeof(int64_t) * (p->m + 1)));
        TRY(dev_alloc(h, h->rowptr, sizeof(int64_t) * (p->m + 1)));
        TRY(dev_alloc(h, h->csr_col, sizeof(int32_t) * nnz));
        TRY(dev_alloc(h, h->csr_val, sizeof(double) * nnz));
        Dev iota, bad;
        TRY(dev_alloc(h, iota, sizeof(int32_t) * nnz));
        TRY(dev_alloc(h, bad, sizeof(unsigned long long)));
        CK(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(counts.p, 0, sizeof(int64_t) * (p->m + 1), h->stream));
        if (p->nnz > 0) {
            expand_colids_kernel<<<grid_for(p->n, 256, 8 * h->sms), 256, 0, h->stream>>>(P_<int64_t>(h->colptr), p->n,
                                                                                          P_<int32_t>(colid));
            CKL();
            iota_kernel<<<grid_for(p->nnz, 256, 8 * h->sms), 256, 0, h->stream>>>(P_<int32_t>(iota), p->nnz);
            CKL();
            row_count_kernel<<<grid_for(p->nnz, 256, 8 * h->sms), 256, 0, h->stream>>>(
                P_<int32_t>(h->rowidx), p->nnz, p->m, P_<int64_t>(counts), P_<unsigned long long>(bad));
            CKL();
            size_t tmp_bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, P_<int32_t>(h->rowidx), P_<int32_t>(keys_out),
                                            P_<int32_t>(iota), P_<int32_t>(perm), (int)p->nnz, 0, 32, h->stream);
            Dev tmp;
            TRY(dev_alloc(h, tmp, tmp_bytes));
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, P_<int32_t>(h->rowidx), P_<int32_t>(keys_out),
                                               P_<int32_t>(iota), P_<int32_t>(perm), (int)p->nnz, 0, 32, h->stream));
            csr_gather_kernel<<<grid_for(p->nnz, 256, 8 * h->sms), 256, 0, h->stream>>>(
                P_<int32_t>(perm), P_<int32_t>(colid), P_<double>(h->vals), p->nnz, P_<int32_t>(h->csr_col),
                P_<double>(h->csr_val));
            CKL();
            CK(cudaStreamSynchronize(h->stream));
            dev_free(tmp);
        }
        size_t scan_bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, P_<int64_t>(counts), P_<int64_t>(h->rowptr),
                                      (int)(p->m + 1), h->stream);
        Dev scan_tmp;
        TRY(dev_alloc(h, scan_tmp, scan_bytes));
        CK(cub::DeviceScan::ExclusiveSum(scan_tmp.p, scan_bytes, P_<int64_t>(counts), P_<int64_t>(h->rowptr),
                                         (int)(p->m + 1), h->stream));
        unsigned long long nbad = 0;
        CK(cudaMemcpyAsync(&nbad, bad.p, sizeof nbad, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        Dev* tmps[] = {&colid, &perm, &keys_out, &counts, &iota, &bad, &scan_tmp};
        for (Dev* d : tmps) dev_free(*d);
        if (nbad) {
            free_problem(h);
            return h->fail(ASY_ERR_INVALID, "rowidx has %llu entries outside [0, m)", nbad);
        }
    }

    // ---- vectors
    TRY(dev_alloc(h, h->b, sizeof(double) * (p->m + 32)));  // padded: bulk copies of b rows
    CK(cudaMemsetAsync(h->b.p, 0, sizeof(double) * (p->m + 32), h->stream));
    CK(cudaMemcpyAsync(h->b.p, p->b, sizeof(double) * p->m,
                       cm == ASY_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
    TRY(copy_in(h, h->tau, p->tau, sizeof(double) * p->n, cm));
    if (p->lo) {
        TRY(copy_in(h, h->lo, p->lo, sizeof(double) * p->n, cm));
        TRY(copy_in(h, h->hi, p->hi, sizeof(double) * p->n, cm));
    }
    // validate tau / box
    {
        Dev bad;
        TRY(dev_alloc(h, bad, sizeof(unsigned long long)));
        CK(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), h->stream));
        validate_kernel<<<grid_for(p->n, 256, 4 * h->sms), 256, 0, h->stream>>>(
            P_<double>(h->tau), p->lo ? P_<double>(h->lo) : nullptr, p->hi ? P_<double>(h->hi) : nullptr, p->n,
            P_<unsigned long long>(bad));
        CKL();
        unsigned long long nbad = 0;
        CK(cudaMemcpyAsync(&nbad, bad.p, sizeof nbad, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        dev_free(bad);
        if (nbad) {
            free_problem(h);
            return h->fail(ASY_ERR_INVALID, "%llu coordinates with tau <= 0 (or inf/nan) or lo > hi", nbad);
        }
    }

    // ---- scalars
    Scalars& S = h->S;
    S = Scalars{};
    S.loss = p->loss;
    S.reg = p->reg;
    S.s2 = 2.0 * p->loss_scale;
    S.minv = 1.0 / (double)p->m;
    S.c2 = 2.0 * p->c_nonconvex;
    S.lam = p->lambda;
    S.theta = p->theta;
    if (p->reg == ASY_REG_EXP) S.eta = p->theta;
    else if (p->reg == ASY_REG_LOG) S.eta = p->theta / log1p(p->theta);
    else S.eta = 1.0;
    S.inv_log1p_theta = p->reg == ASY_REG_LOG ? 1.0 / log1p(p->theta) : 0.0;
    S.lam_eff = p->reg == ASY_REG_L1 ? p->lambda : p->lambda * S.eta;
    S.lo_all = p->lo_all;
    S.hi_all = p->hi_all;
    S.lo = p->lo ? P_<double>(h->lo) : nullptr;
    S.hi = p->hi ? P_<double>(h->hi) : nullptr;

    // ---- state
    TRY(dev_alloc(h, h->x, sizeof(double) * h->n));
    TRY(dev_alloc(h, h->xalt, sizeof(double) * h->n));
    TRY(dev_alloc(h, h->xs, sizeof(double) * h->n));
    TRY(dev_alloc(h, h->dx, sizeof(double) * h->n));
    TRY(dev_alloc(h, h->mf, sizeof(double) * h->n));
    TRY(dev_alloc(h, h->mer, sizeof(double) * h->n));
    TRY(dev_alloc(h, h->r, sizeof(double) * (h->m + 32)));  // padded: bulk copies of residual rows
    TRY(dev_alloc(h, h->rs, sizeof(double) * h->m));
    TRY(dev_alloc(h, h->w, sizeof(double) * (h->m + 2)));
    h->has_problem = true;
    TRY(reset_state(h, nullptr, ASY_MEM_DEVICE));
    CK(cudaStreamSynchronize(h->stream));
    return ASY_OK;
}

// ---- one synchronous Jacobi sweep
static int jacobi_sweep(asy_handle* h, double gamma) {
    loss_weights_kernel<<<grid_for(h->m, 256, 4 * h->sms), 256, 0, h->stream>>>(h->S, P_<double>(h->r),
                                                                                  P_<double>(h->b), P_<double>(h->w), h->m);
    CKL();
    TRY(gemvT(h, P_<double>(h->w), GT_JACOBI, P_<double>(h->x), gamma, P_<double>(h->dx), nullptr, nullptr));
    TRY(gemvN(h, P_<double>(h->dx), COMBINE_ADD, P_<double>(h->r)));
    return ASY_OK;
}

// ---- async launches
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

struct DenseGeom {
    int64_t R, G, delay;
    int Bpad, grid, use_tmem, too_tall = 0;
    size_t smem;
    const void* kernel;
};

// compiled (BT, RPL) instantiations of dense_async_kernel: BT = block width padded to
// {8,16,32,64,128}, RPL = panel rows per lane; default R*BT = 4096 doubles (32 KB panels)
using DenseKernelFn = void (*)(const CUtensorMap, const DenseAsyncParams);
static DenseKernelFn dense_kernel_for(int BT, int RPL, int NS, int loss) {
#define ASY_DK(bt, rpl, ns)                                                                   \
    if (BT == bt && RPL == rpl && NS == ns)                                                   \
        return loss == LOSS_LS ? dense_async_kernel<bt, rpl, ns, LOSS_LS>                     \
                               : dense_async_kernel<bt, rpl, ns, LOSS_LOGISTIC>;
    ASY_DK(8, 8, 4) ASY_DK(16, 8, 4) ASY_DK(32, 4, 4) ASY_DK(32, 3, 8) ASY_DK(32, 2, 8) ASY_DK(64, 2, 4) ASY_DK(128, 1, 4)
#undef ASY_DK
    return nullptr;
}

static int dense_geometry(asy_handle* h, const asy_solve_params* sp, int64_t delay, DenseGeom* g) {
    const int64_t B = h->B;
    int BT = 8;
    while (BT < B) BT *= 2;
    // (measured on configs 1-3: one 32 KB stage per pair beats two smaller ones -- the
    // per-panel fixed costs dominate, not the load latency)
    int RPL = BT == 8 ? 8 : BT == 16 ? 8 : BT == 32 ? 4 : BT == 64 ? 2 : 1;
    int NS = kPairs;
    if (dbg_env("ASY_DENSE_RPL")) RPL = atoi(dbg_env("ASY_DENSE_RPL"));
    if (dbg_env("ASY_DENSE_NS")) NS = atoi(dbg_env("ASY_DENSE_NS"));
    // requested panel rows / stages: honoured when that (BT, RPL, NS) kernel is compiled, refused otherwise
    if (sp->panel_rows > 0) RPL = sp->panel_rows / 32;
    if (sp->stages > 0) NS = sp->stages;
    else if (sp->panel_rows > 0 && !dense_kernel_for(BT, RPL, NS, h->S.loss) &&
             dense_kernel_for(BT, RPL, 2 * kPairs, h->S.loss))
        NS = 2 * kPairs;  // (only the rows were asked for: the stage count compiled for them)
    const int64_t R = 32 * RPL;
    const int64_t G = (h->m + R - 1) / R;
    DenseKernelFn fn = dense_kernel_for(BT, RPL, NS, h->S.loss);
    if (!fn)
        return h->fail(ASY_ERR_UNSUPPORTED, "panel kernel: no compiled geometry for %d-column blocks with %d panel rows "
                       "and %d stages", BT, 32 * RPL, NS);
    int use_tmem = RPL * 2 * BT <= kSlotCols;
    if (tuning_of(sp).panel_park == 2) use_tmem = 0;  // re-read panels from L2 instead of parking them
    constexpr int NAX = kPairs * kAxpyPerPair;
    const size_t smem = sizeof(double) * (NS * (R * BT + 2 * R) + NAX * BT) +
                        sizeof(StageMeta) * (NS + kQueue) + sizeof(Handoff) * NAX * kRing +
                        sizeof(uint64_t) * (2 * NS + 2 * kQueue + 2 * NAX * kRing) + sizeof(unsigned) * (NAX + 1) +
                        64;
    if (smem > 227 * 1024)
        return h->fail(ASY_ERR_INVALID, "panel_rows*block_size too large for shared memory (%zu B)", smem);
    CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, kDenseThreads, smem));
    if (occ < 1) return h->fail(ASY_ERR_CUDA, "dense async kernel does not fit on an SM");
    int grid = h->sms;  // one CTA per SM: it owns the SM's whole TMEM (512 columns)
    // enough workers to keep ~2x the delay window of panels in flight, never more
    const int64_t want = (2 * (delay + 1) * G + kPairs - 1) / kPairs;
    if (want < grid) grid = (int)std::max<int64_t>(1, want);
    if (sp->workers > 0) grid = std::min(grid, (int)sp->workers);
    // Every panel of a block must be published (handed off) before the block's solve can run, so
    // the G panels of one block must fit in a quarter of the hand-off rings of the workers
    // (kRing notes per axpy warp); otherwise a full ring would stall a dot warp that holds its
    // smem stage while panels of the same block wait for that stage (deadlock).  Such shapes
    // (very tall blocks on few workers) go to the row-slab kernel instead.
    if (4 * G > (int64_t)kRing * NAX * grid) {
        g->too_tall = 1;
        return h->fail(ASY_ERR_UNSUPPORTED, "panel kernel: %lld panels per block exceed the hand-off capacity of "
                       "%d workers", (long long)G, grid);
    }
    // blocks in flight are capped so that a block's panels never fill an axpy warp's hand-off ring
    const int64_t cap = std::max<int64_t>(0, (int64_t)kRing * NAX * grid / (4 * G) - 1);
    g->delay = std::min<int64_t>(delay, cap);
    g->R = R; g->G = G; g->Bpad = BT; g->grid = grid; g->smem = smem; g->use_tmem = use_tmem;
    g->kernel = (const void*)fn;
    return ASY_OK;
}

#ifndef ASY_LGW_MAX
#define ASY_LGW_MAX 3  // D1 windows of at most 8 sequences
#endif
static int dense_async_launch(asy_handle* h, const asy_solve_params* sp, int64_t sweeps, int64_t delay,
                              float* ms, bool* too_tall) {
    DenseGeom geo;
    const int grc = dense_geometry(h, sp, delay, &geo);
    if (grc != ASY_OK) {
        if (too_tall) *too_tall = geo.too_tall != 0;
        return grc;
    }
    const int64_t B = h->B, R = geo.R, G = geo.G;
    const int Bmax = (int)B;
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return h->fail(ASY_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmap;
    cuuint64_t dims[2] = {(cuuint64_t)h->m, (cuuint64_t)h->n};
    cuuint64_t strides[1] = {(cuuint64_t)(h->lda * sizeof(double))};
    cuuint32_t box[2] = {(cuuint32_t)R, (cuuint32_t)geo.Bpad};  // BT columns (extra ones are OOB zeros / ignored)
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->A.p, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return h->fail(ASY_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
    const int64_t slots = next_pow2(std::max<int64_t>(1024, 2 * (delay + 2)));
    TRY(dev_alloc(h, h->gacc, sizeof(double) * 2 * slots * kPanelRep * Bmax));
    TRY(dev_alloc(h, h->dpart, sizeof(double) * G * Bmax));
    TRY(dev_alloc(h, h->arrive, sizeof(unsigned) * slots * kCtrPad));
    TRY(dev_alloc(h, h->consumed, sizeof(unsigned) * slots * kCtrPad));
    TRY(dev_alloc(h, h->ver, sizeof(unsigned) * h->nblk * kCtrPad));
    // D1 windows: W <= delay + 1 sequences (the windows a sequence waits for end before it),
    // SW > (delay + 2) / W + 2 slots (a window slot is reused only after its window completed)
    const int64_t geo_delay = geo.delay;
    int lg_w = 0;
    while (lg_w < ASY_LGW_MAX && ((int64_t)2 << lg_w) <= (geo_delay + 1) / 4) ++lg_w;  // (W <= (delay + 1) / 4)
    const int64_t wslots = next_pow2(std::max<int64_t>(64, ((geo_delay + 2) >> lg_w) + 8));
    int lg_sw = 0;
    while (((int64_t)1 << lg_sw) < wslots) ++lg_sw;
    TRY(dev_alloc(h, h->wcnt, sizeof(unsigned) * wslots * kCtrPad));

    DenseAsyncParams P{};
    P.A = P_<double>(h->A); P.lda = h->lda;
    // a block whose panels exceed ~half the machine's TMEM slots will be partly re-read: keep it in L2
    P.keep_in_l2 = !geo.use_tmem || G * 2 > (int64_t)geo.grid * kPairs * kTmemSlots;
    P.m = h->m; P.n = h->n; P.B = B; P.nblk = h->nblk; P.R = R; P.G = G; P.use_tmem = geo.use_tmem;
    // claims of 2 subtasks for narrow blocks (measured +4% on configs[1]), 4 otherwise (configs[2])
    P.claim = geo.Bpad <= 32 ? 2 : kClaim;
    // cyclic schedule with delay < N - 1: a block's previous update (sequence k - N) is covered by
    // the D1 watermark's acquire; otherwise the D4 loads acquire themselves
    P.wcnt = P_<unsigned>(h->wcnt); P.lg_w = lg_w; P.lg_sw = lg_sw;
    P.measure_delay = tuning_of(sp).measure_delay != 0;
    if (const char* e = dbg_env("ASY_CLAIM_N")) P.claim = std::max(1, std::min(kClaim, atoi(e)));
    P.r = P_<double>(h->r); P.aux = P_<double>(h->b); P.tau = P_<double>(h->tau);
    P.x0 = P_<double>(h->x); P.x1 = P_<double>(h->xalt);
    P.S = h->S; P.gamma = sp->gamma; P.sched = sp->schedule; P.seed = sp->seed; P.epoch0 = h->epochs;
    delay = geo.delay;
    h->last_kernel = ASY_KERNEL_DENSE_PANEL;
    h->last_delay = (int)delay;
    P.T = sweeps * h->nblk * G; P.delay = delay; P.deterministic = delay == 0 ? 1 : 0;
    P.counter = P_<unsigned long long>(h->counter); P.gacc = P_<double>(h->gacc);
    P.part = P_<double>(h->dpart); P.arrive = P_<unsigned>(h->arrive); P.consumed = P_<unsigned>(h->consumed);
    P.xver = P_<unsigned>(h->ver);
    P.slots = slots; P.Bmax = Bmax; P.Bpad = geo.Bpad;
    TRY(dev_alloc(h, h->dobs, sizeof(unsigned)));
    CK(cudaMemsetAsync(h->dobs.p, 0, sizeof(unsigned), h->stream));
    P.dobs = P_<unsigned>(h->dobs);
    P.lg_slots = 0;
    while (((int64_t)1 << P.lg_slots) < slots) ++P.lg_slots;

    // debug trace (env ASY_TRACE=<subtasks>, ASY_TRACE_FILE=<path>): globaltimer stamps per subtask
    const char* tr = dbg_env("ASY_TRACE");
    Dev trace;
    if (tr && atoll(tr) > 0) {
        P.trace_n = std::min<int64_t>(atoll(tr), P.T);
        TRY(dev_alloc(h, trace, sizeof(unsigned long long) * 12 * P.trace_n));
        CK(cudaMemsetAsync(trace.p, 0, sizeof(unsigned long long) * 12 * P.trace_n, h->stream));
        P.trace = P_<unsigned long long>(trace);
    }
    const char* pf = dbg_env("ASY_PROF");
    Dev prof;
    if (pf) {
        TRY(dev_alloc(h, prof, sizeof(unsigned long long) * geo.grid * 16 * 8));
        CK(cudaMemsetAsync(prof.p, 0, sizeof(unsigned long long) * geo.grid * 16 * 8, h->stream));
        P.prof = P_<unsigned long long>(prof);
    }
    dense_async_init<<<grid_for(std::max<int64_t>(2 * slots * kPanelRep * Bmax, h->nblk), 256, 4 * h->sms), 256, 0, h->stream>>>(P);
    CKL();
    void* args[] = {&tmap, &P};
    CK(cudaEventRecord(h->ev[0], h->stream));
    CK(cudaLaunchCooperativeKernel(geo.kernel, dim3(geo.grid), dim3(kDenseThreads), args, geo.smem, h->stream));
    CK(cudaEventRecord(h->ev[1], h->stream));
    CK(cudaEventSynchronize(h->ev[1]));
    CKL();
    CK(cudaEventElapsedTime(ms, h->ev[0], h->ev[1]));
    if (P.measure_delay) {
        unsigned dobs = 0;
        CK(cudaMemcpy(&dobs, h->dobs.p, sizeof(unsigned), cudaMemcpyDeviceToHost));
        h->last_dobs = std::max(h->last_dobs, (int)dobs);
    }
    if (sweeps & 1) std::swap(h->x, h->xalt);  // the updated iterate lives in the other half
    if (P.prof) {
        std::vector<unsigned long long> hb((size_t)geo.grid * 16 * 8);
        CK(cudaMemcpy(hb.data(), prof.p, sizeof(unsigned long long) * hb.size(), cudaMemcpyDeviceToHost));
        FILE* f = fopen(pf, "wb");
        if (f) {
            fwrite(hb.data(), sizeof(unsigned long long), hb.size(), f);
            fclose(f);
        }
        dev_free(prof);
    }
    if (P.trace) {
        std::vector<unsigned long long> hb(12 * P.trace_n);
        CK(cudaMemcpy(hb.data(), trace.p, sizeof(unsigned long long) * hb.size(), cudaMemcpyDeviceToHost));
        const char* fn = dbg_env("ASY_TRACE_FILE");
        FILE* f = fopen(fn ? fn : "asy_trace.bin", "wb");
        if (f) {
            fwrite(hb.data(), sizeof(unsigned long long), hb.size(), f);
            fclose(f);
        }
        dev_free(trace);
    }
    return ASY_OK;
}

// ---- row-slab dense async kernel (dense_slab.cuh)
using SlabKernelFn = void (*)(const CUtensorMap, const SlabParams);
static SlabKernelFn slab_kernel_for(int cpw, int loss) {
    if (loss == LOSS_LS) {
        if (cpw == 8) return dense_slab_kernel<8, LOSS_LS>;
        if (cpw == 16) return dense_slab_kernel<16, LOSS_LS>;
        if (cpw == 32) return dense_slab_kernel<32, LOSS_LS>;
    } else {
        if (cpw == 8) return dense_slab_kernel<8, LOSS_LOGISTIC>;
        if (cpw == 16) return dense_slab_kernel<16, LOSS_LOGISTIC>;
        if (cpw == 32) return dense_slab_kernel<32, LOSS_LOGISTIC>;
    }
    return nullptr;
}

// ---- row-slab kernel with the tile parked in TMEM (dense_slabt.cuh)
static SlabKernelFn slabt_kernel_for(int bmax, int cs, int loss) {
    if (loss == LOSS_LS) {
        if (bmax == 32) return dense_slabt_kernel<32, LOSS_LS>;
        if (bmax == 64) return cs == 64 ? dense_slabt_kernel<64, LOSS_LS, 64> : dense_slabt_kernel<64, LOSS_LS>;
        if (bmax == 128) return dense_slabt_kernel<128, LOSS_LS>;
    } else {
        if (bmax == 32) return dense_slabt_kernel<32, LOSS_LOGISTIC>;
        if (bmax == 64) return cs == 64 ? dense_slabt_kernel<64, LOSS_LOGISTIC, 64> : dense_slabt_kernel<64, LOSS_LOGISTIC>;
        if (bmax == 128) return dense_slabt_kernel<128, LOSS_LOGISTIC>;
    }
    return nullptr;
}

// Geometry of the TMEM-parking slab kernel (dense_slabt.cuh); false when its park ring
// (TMEM + shared-memory hold slots: one whole sequence per dot warp) plus a load ring of
// >= 4 units per dot warp does not fit on the SM, or a warp would own > kSlabTMaxG groups.
struct SlabTGeom {
    int grid, bmax, nsw, nhold, npark[4], hoff[4], rotate, cs;
    int64_t Rs;
    size_t smem;
};
static bool slabt_geometry(const asy_handle* h, const asy_solve_params* sp, SlabTGeom* g) {
    const int64_t m = h->m, B = h->B;
    if (B > 128) return false;
    const int bmax = B <= 32 ? 32 : B <= 64 ? 64 : 128;
    // sub-sequence width: 32 columns (blocks of 65-128: four all-reduces per update overlap the
    // later columns' loads), the whole block for blocks of 33-64 (one all-reduce per update)
    int cs = bmax == 64 ? 64 : 32;
    if (const char* e = dbg_env("ASY_SLABT_CS")) cs = (atoi(e) == 64 && bmax == 64) ? 64 : 32;
    const int CS = cs, nsplit = bmax / CS, SQ = 256 / CS;
    g->cs = cs;
    // slabs of whole 32-row groups: ngt groups over the CTAs, ngt / grid or one more each
    const int64_t ngt = (m + 31) / 32;
    int64_t grid0 = h->sms;
    if (sp->workers > 0) grid0 = std::min<int64_t>(grid0, sp->workers);
    grid0 = std::max<int64_t>(1, std::min<int64_t>(grid0, ngt));
    const int nrg = (int)((ngt + grid0 - 1) / grid0);  // most groups of a CTA
    const int64_t Rs = 32 * (int64_t)nrg;
    if ((nrg + kSlabDot - 1) / kSlabDot > kSlabTMaxG) return false;
    const int UC = std::min(kSlabTUnitCols, CS);  // unit columns (dense_slabt.cuh)
    const size_t unit = sizeof(double) * 32 * UC, hslot = sizeof(double) * 32 * CS;
    const int64_t RsP = (Rs + 1) & ~1ll;
    const size_t fixed = sizeof(double) * (3 * RsP + kSlabDot * kSlabTMaxG * 32 + (size_t)(kSlabNP * kSlabDot + kSlabNDX) * CS) +
                         (sizeof(SeqMeta) + sizeof(long long)) * kSlabNM +
                         sizeof(uint64_t) * (2 * kSlabTMaxStages + 2 * kSlabNP + 3 * kSlabNDX) +
                         sizeof(unsigned long long) * (kSlabAx + kSlabDot) + sizeof(unsigned) * (kSlabDot + 1) + 256;
    const size_t cap = 227 * 1024;
    // park ring of dot warp d: np slots (TMEM first, then shared-memory hold slots), at least the
    // nsplit sub-sequences of one block update for each of its groups (deadlock freedom); with
    // more, the warp may start a sub-sequence while the all-reduces of earlier ones are in flight
    // the last, partial round of groups rotates over the warps (any warp may hold one of them)
    g->rotate = 1;
    if (const char* e = dbg_env("ASY_SLABT_ROTATE")) g->rotate = atoi(e) != 0;
    // Shared memory is split between the load rings (nsw unit stages per dot warp) and the hold
    // slots that deepen the park rings beyond TMEM.  Both matter: the park ring must cover the
    // all-reduce chain (~2 block updates of latency), the load ring the HBM latency.  Measured
    // on configs[2] (np / nsw): 4 / 12 4.27, 5 / 8 4.51, 5 / 6 4.56, 6 / 4 4.06 TB/s; on configs[3]:
    // 8 / 12 4.2, 9 / 10 4.93, 10 / 8 5.04, 11 / 6 5.14, 12 / 4 5.03.  Rule: the deepest park ring
    // (at most 3 spare sub-sequences) that leaves >= 6 stages per warp, else >= 4 stages.
    int nsw = 0, nhold = 0;
    int ring = tuning_of(sp).slab_ring;  // (test / measurement override of the ring depth)
    if (const char* e = dbg_env("ASY_SLABT_RING")) ring = atoi(e);
    const int per4k = UC / 16;  // 4 KB per unit stage
    const int min_first = ring > 0 ? ring : std::max(2, 6 / per4k), min_last = ring > 0 ? min_first : std::max(1, 4 / per4k);
    int cntmax = 0;
    for (int d = 0; d < kSlabDot; ++d)
        cntmax = std::max(cntmax, g->rotate ? nrg / kSlabDot + (nrg % kSlabDot ? 1 : 0)
                                            : (nrg > d ? (nrg - d + kSlabDot - 1) / kSlabDot : 0));
    // (deadlock freedom needs only one sub-sequence's slots, np >= cntmax: sub-sequence (k, h) then
    // waits for the axpy of (k, h - 1), whose all-reduce needs no CTA to go beyond (k, h - 1))
    int np_hi = (nsplit + 3) * cntmax, np_lo = cntmax;  // park slots of the busiest warp
    if (const char* e = dbg_env("ASY_SLABT_NPARK")) np_hi = np_lo = std::max(np_lo, atoi(e));
    for (int min_nsw = min_first; min_nsw >= min_last && nsw == 0; min_nsw -= std::max(1, 2 / per4k))
    for (int np = np_hi; np >= np_lo; --np) {
        nhold = 0;
        for (int d = 0; d < kSlabDot; ++d) {
            const int cnt = g->rotate ? nrg / kSlabDot + (nrg % kSlabDot ? 1 : 0)
                                      : (nrg > d ? (nrg - d + kSlabDot - 1) / kSlabDot : 0);
            // a warp with fewer groups keeps the same depth in block updates
            const int want = cnt == cntmax ? np : std::max(cnt, (np * cnt + cntmax - 1) / cntmax);
            const int hs = std::max(0, want - SQ);
            g->hoff[d] = nhold;
            g->npark[d] = SQ + hs;
            nhold += hs;
        }
        nsw = kSlabTMaxStages / kSlabDot;
        if (ring > 0) nsw = std::max(1, std::min(nsw, ring));
        while (nsw > min_nsw && fixed + nhold * hslot + kSlabDot * nsw * unit > cap) --nsw;
        // (an odd ring of 4 KB units halves the issuing lanes: -25%; 8 KB boxes need only one lane per ring)
        if (per4k == 1 && ring <= 0 && nsw > min_nsw && (nsw & 1)) --nsw;
        if (nsw >= min_nsw && fixed + nhold * hslot + kSlabDot * nsw * unit <= cap) break;
        nsw = 0;
    }
    if (nsw == 0) return false;
    g->grid = (int)grid0;
    g->Rs = Rs; g->bmax = bmax; g->nsw = nsw; g->nhold = nhold;
    g->smem = fixed + nhold * hslot + kSlabDot * nsw * unit;
    return true;
}

static int dense_slabt_launch(asy_handle* h, const asy_solve_params* sp, const SlabTGeom& geo, int64_t sweeps,
                              int64_t delay, float* ms) {
    const int64_t B = h->B;
    delay = std::min<int64_t>(delay, kSlabNM - 64);  // metadata ring depth
    const int nsplit = geo.bmax / geo.cs;  // all-reduces per block update
    const int64_t slots = next_pow2(std::max<int64_t>(64, nsplit * (2 * delay + 2)));
    const int det = delay == 0 ? 1 : 0;
    h->last_kernel = ASY_KERNEL_DENSE_SLAB_TMEM;
    h->last_delay = (int)delay;
    SlabKernelFn fn = slabt_kernel_for(geo.bmax, geo.cs, h->S.loss);
    if (!fn) return h->fail(ASY_ERR_UNSUPPORTED, "no TMEM slab kernel for block size %lld", (long long)B);
    CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)geo.smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, kSlabThreads, geo.smem));
    if (occ < 1) return h->fail(ASY_ERR_CUDA, "TMEM slab kernel does not fit on an SM");

    EncodeTiledFn enc = encode_tiled();
    if (!enc) return h->fail(ASY_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmap;
    const int UCk = std::min(kSlabTUnitCols, geo.cs);
    const int W = B < UCk ? (int)B : UCk;  // unit box: 32 rows x UC columns
    cuuint64_t dims[2] = {(cuuint64_t)h->m, (cuuint64_t)h->n};
    cuuint64_t strides[1] = {(cuuint64_t)(h->lda * sizeof(double))};
    cuuint32_t box[2] = {32u, (cuuint32_t)W};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->A.p, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return h->fail(ASY_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);

    TRY(dev_alloc(h, h->gacc, sizeof(double) * 2 * slots * kGaccRep * B));
    TRY(dev_alloc(h, h->arrive, sizeof(unsigned) * slots * kArrivePad));
    if (det) TRY(dev_alloc(h, h->dpart, sizeof(double) * slots * geo.grid * B));

    SlabParams P{};
    P.m = h->m; P.n = h->n; P.B = B; P.nblk = h->nblk;
    P.Rs = geo.Rs; P.Rc = 32; P.nch = (int)((geo.Rs + 31) / 32); P.hold = 1;
    P.nst = kSlabDot * geo.nsw; P.nsa = geo.nhold; P.stage_dbl = 32 * UCk;
    P.r = P_<double>(h->r); P.aux = P_<double>(h->b); P.tau = P_<double>(h->tau);
    P.x0 = P_<double>(h->x); P.x1 = P_<double>(h->xalt);
    P.S = h->S; P.gamma = sp->gamma; P.sched = sp->schedule; P.seed = sp->seed; P.epoch0 = h->epochs;
    P.K = sweeps * h->nblk; P.delay = delay; P.deterministic = det;
    P.gacc = P_<double>(h->gacc); P.part = det ? P_<double>(h->dpart) : nullptr; P.arrive = P_<unsigned>(h->arrive);
    P.slots = slots;
    P.A = P_<double>(h->A); P.lda = h->lda;
    for (int d = 0; d < 4; ++d) { P.npark[d] = geo.npark[d]; P.hoff[d] = geo.hoff[d]; }
    P.rotate = geo.rotate;
    TRY(dev_alloc(h, h->dobs, sizeof(unsigned)));
    CK(cudaMemsetAsync(h->dobs.p, 0, sizeof(unsigned), h->stream));
    P.dobs = P_<unsigned>(h->dobs);
    const char* pf = dbg_env("ASY_PROF");
    Dev prof;
    if (pf) {
        TRY(dev_alloc(h, prof, sizeof(unsigned long long) * geo.grid * kSlabWarps * 8));
        CK(cudaMemsetAsync(prof.p, 0, sizeof(unsigned long long) * geo.grid * kSlabWarps * 8, h->stream));
        P.prof = P_<unsigned long long>(prof);
    }
    if (dbg_env("ASY_SLAB_VERBOSE"))
        fprintf(stderr, "[slabt] grid %d Rs %lld bmax %d nsw %d nhold %d npark %d/%d/%d/%d smem %zu delay %lld det %d\n",
                geo.grid, (long long)geo.Rs, geo.bmax, geo.nsw, geo.nhold, geo.npark[0], geo.npark[1], geo.npark[2],
                geo.npark[3], geo.smem, (long long)delay, det);
    slab_init<<<grid_for(2 * slots * kGaccRep * B, 256, 4 * h->sms), 256, 0, h->stream>>>(P);
    CKL();
    void* args[] = {&tmap, &P};
    CK(cudaEventRecord(h->ev[0], h->stream));
    CK(cudaLaunchCooperativeKernel((const void*)fn, dim3(geo.grid), dim3(kSlabThreads), args, geo.smem, h->stream));
    CK(cudaEventRecord(h->ev[1], h->stream));
    CK(cudaEventSynchronize(h->ev[1]));
    CKL();
    CK(cudaEventElapsedTime(ms, h->ev[0], h->ev[1]));
    {
        unsigned dobs = 0;
        CK(cudaMemcpy(&dobs, h->dobs.p, sizeof(unsigned), cudaMemcpyDeviceToHost));
        h->last_dobs = std::max(h->last_dobs, (int)dobs);
    }
    if (sweeps & 1) std::swap(h->x, h->xalt);
    if (P.prof) {
        std::vector<unsigned long long> hb((size_t)geo.grid * kSlabWarps * 8);
        CK(cudaMemcpy(hb.data(), prof.p, sizeof(unsigned long long) * hb.size(), cudaMemcpyDeviceToHost));
        FILE* f = fopen(pf, "wb");
        if (f) {
            fwrite(hb.data(), sizeof(unsigned long long), hb.size(), f);
            fclose(f);
        }
        dev_free(prof);
    }
    return ASY_OK;
}

static int dense_slab_launch(asy_handle* h, const asy_solve_params* sp, int64_t sweeps, int64_t delay, float* ms) {
    {
        // the TMEM-parking form when its park ring fits (ASY_SLAB_TMEM=0: the smem / L2 form)
        SlabTGeom tg;
        if (tuning_of(sp).dense_kernel != ASY_KERNEL_DENSE_SLAB && slabt_geometry(h, sp, &tg))
            return dense_slabt_launch(h, sp, tg, sweeps, delay, ms);
    }
    const int64_t m = h->m, B = h->B;
    const int cpw = B <= 32 ? 8 : B <= 64 ? 16 : 32;
    const int BMAX = kSlabDot * cpw;
    if (B > BMAX) return h->fail(ASY_ERR_UNSUPPORTED, "block size %lld > %d", (long long)B, BMAX);
    // slabs: one CTA per SM, at least 16 rows each, every CTA owns >= 1 row
    int64_t grid0 = h->sms;
    if (sp->workers > 0) grid0 = std::min<int64_t>(grid0, sp->workers);
    grid0 = std::max<int64_t>(1, std::min<int64_t>(grid0, (m + 15) / 16));
    int64_t Rs = (m + grid0 - 1) / grid0;
    Rs += Rs & 1;  // even: 16-byte aligned TMA row starts
    const int grid = (int)((m + Rs - 1) / Rs);
    // chunks of Rc rows (TMA box Rc x B, Rc even, <= 256): fewest rows loaded past the slab,
    // then fewest chunks, with stages of at most ~24 KB (ASY_SLAB_CHUNK_KB)
    int nch = 0, Rc = 0;
    {
        const char* ckb = dbg_env("ASY_SLAB_CHUNK_KB");
        const int64_t chunk_bytes = 1024 * (ckb ? std::max(1, atoi(ckb)) : 24);
        const int64_t max_rows = std::max<int64_t>(2, std::min<int64_t>(256, (chunk_bytes / (8 * BMAX)) & ~1ll));
        int64_t best_waste = -1;
        const int64_t n0 = (Rs + max_rows - 1) / max_rows;
        for (int64_t c = n0; c <= n0 + 4; ++c) {
            int64_t rc = (Rs + c - 1) / c;
            rc += rc & 1;
            if (rc > max_rows) continue;
            const int64_t waste = c * rc - Rs;
            if (best_waste < 0 || waste < best_waste) { best_waste = waste; nch = (int)c; Rc = (int)rc; }
        }
        if (const int rc = tuning_of(sp).slab_chunk_rows) {  // (test override)
            Rc = std::max(2, std::min(256, rc & ~1));
            nch = (int)((Rs + Rc - 1) / Rc);
        }
    }
    const int64_t RsP = (Rs + 1) & ~1ll;
    const int64_t stage_dbl = ((int64_t)Rc * BMAX + kSlabPad + 15) & ~15ll;
    const size_t stage_bytes = sizeof(double) * stage_dbl;
    const size_t fixed = sizeof(double) * (2 * RsP + (size_t)(kSlabNP * kSlabDot + kSlabNDX) * BMAX + kSlabDot * 256) +
                         sizeof(SeqMeta) * kSlabNM +
                         sizeof(uint64_t) * (4 * kSlabMaxStages + 2 * kSlabNP + 2 * kSlabNDX) +
                         sizeof(unsigned long long) * (kSlabAx + kSlabDot) + 128;
    const size_t cap = 227 * 1024;
    if (fixed + 3 * stage_bytes > cap) return h->fail(ASY_ERR_UNSUPPORTED, "row slab too tall for shared memory");
    int total = (int)std::min<size_t>((cap - fixed) / stage_bytes, 2 * kSlabMaxStages);
    // dot stages come in per-dot-warp sub-rings (kSlabDot of them).  Hold the chunks until
    // the axpy when >= 2 sequences per dot warp fit, else re-load them from L2.
    int hold = total / kSlabDot >= 2 * nch;
    if (const int hv = tuning_of(sp).slab_hold) hold = hv == 1 && total / kSlabDot >= nch + 1;
    int nst, nsa;
    if (hold) {
        nst = std::min(total, kSlabMaxStages) / kSlabDot * kSlabDot;
        nsa = 0;
    } else {
        nsa = std::max(1, std::min(nch, total - kSlabDot));
        if (total - nsa >= 2 * kSlabDot && nsa > 2) nsa = 2;
        nst = std::min(total - nsa, kSlabMaxStages) / kSlabDot * kSlabDot;
    }
    if (nst < kSlabDot || (!hold && nsa < 1))
        return h->fail(ASY_ERR_UNSUPPORTED, "row slab chunks too large for shared memory");
    const size_t smem = fixed + stage_bytes * (nst + nsa);
    // delay: the L2 must still hold a block between its dot pass and its re-load
    if (!hold) {
        const double blk_bytes = 8.0 * (double)m * (double)B;
        const char* l2e = dbg_env("ASY_SLAB_L2MB");  // measurement override of the L2 budget
        const double l2b = (l2e ? atof(l2e) : 40.0) * 1e6;
        const int64_t l2cap = std::max<int64_t>(1, (int64_t)(l2b / blk_bytes));
        delay = std::min(delay, l2cap);
    }
    delay = std::min<int64_t>(delay, kSlabNM - 64);  // metadata ring depth
    const int64_t slots = next_pow2(std::max<int64_t>(64, 2 * delay + 2));
    const int det = delay == 0 ? 1 : 0;
    h->last_kernel = ASY_KERNEL_DENSE_SLAB;
    h->last_delay = (int)delay;

    SlabKernelFn fn = slab_kernel_for(cpw, h->S.loss);
    CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, kSlabThreads, smem));
    if (occ < 1) return h->fail(ASY_ERR_CUDA, "dense slab kernel does not fit on an SM");

    EncodeTiledFn enc = encode_tiled();
    if (!enc) return h->fail(ASY_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmap;
    cuuint64_t dims[2] = {(cuuint64_t)h->m, (cuuint64_t)h->n};
    cuuint64_t strides[1] = {(cuuint64_t)(h->lda * sizeof(double))};
    cuuint32_t box[2] = {(cuuint32_t)Rc, (cuuint32_t)B};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, h->A.p, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return h->fail(ASY_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);

    TRY(dev_alloc(h, h->gacc, sizeof(double) * 2 * slots * kGaccRep * B));
    TRY(dev_alloc(h, h->arrive, sizeof(unsigned) * slots * kArrivePad));
    if (det) TRY(dev_alloc(h, h->dpart, sizeof(double) * slots * grid * B));

    SlabParams P{};
    P.m = h->m; P.n = h->n; P.B = B; P.nblk = h->nblk;
    P.Rs = Rs; P.Rc = Rc; P.nch = nch; P.hold = hold; P.nst = nst; P.nsa = nsa; P.stage_dbl = stage_dbl;
    P.r = P_<double>(h->r); P.aux = P_<double>(h->b); P.tau = P_<double>(h->tau);
    P.x0 = P_<double>(h->x); P.x1 = P_<double>(h->xalt);
    P.S = h->S; P.gamma = sp->gamma; P.sched = sp->schedule; P.seed = sp->seed; P.epoch0 = h->epochs;
    P.K = sweeps * h->nblk; P.delay = delay; P.deterministic = det;
    P.gacc = P_<double>(h->gacc); P.part = det ? P_<double>(h->dpart) : nullptr; P.arrive = P_<unsigned>(h->arrive);
    P.slots = slots;
    const char* pf = dbg_env("ASY_PROF");
    Dev prof;
    if (pf) {
        TRY(dev_alloc(h, prof, sizeof(unsigned long long) * grid * kSlabWarps * 8));
        CK(cudaMemsetAsync(prof.p, 0, sizeof(unsigned long long) * grid * kSlabWarps * 8, h->stream));
        P.prof = P_<unsigned long long>(prof);
    }
    if (dbg_env("ASY_SLAB_VERBOSE"))
        fprintf(stderr, "[slab] grid %d Rs %lld Rc %d nch %d hold %d nst %d nsa %d smem %zu delay %lld slots %lld det %d\n",
                grid, (long long)Rs, Rc, nch, hold, nst, nsa, smem, (long long)delay, (long long)slots, det);
    slab_init<<<grid_for(2 * slots * kGaccRep * B, 256, 4 * h->sms), 256, 0, h->stream>>>(P);
    CKL();
    void* args[] = {&tmap, &P};
    CK(cudaEventRecord(h->ev[0], h->stream));
    CK(cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kSlabThreads), args, smem, h->stream));
    CK(cudaEventRecord(h->ev[1], h->stream));
    CK(cudaEventSynchronize(h->ev[1]));
    CKL();
    CK(cudaEventElapsedTime(ms, h->ev[0], h->ev[1]));
    if (sweeps & 1) std::swap(h->x, h->xalt);  // the updated iterate lives in the other half
    if (P.prof) {
        std::vector<unsigned long long> hb((size_t)grid * kSlabWarps * 8);
        CK(cudaMemcpy(hb.data(), prof.p, sizeof(unsigned long long) * hb.size(), cudaMemcpyDeviceToHost));
        FILE* f = fopen(pf, "wb");
        if (f) {
            fwrite(hb.data(), sizeof(unsigned long long), hb.size(), f);
            fclose(f);
        }
        dev_free(prof);
    }
    return ASY_OK;
}

// Which dense asynchronous kernel: the row-slab kernel when every SM's share of a block
// update is large (>= 64 KB: tall and wide blocks, e.g. configs[2] and [3]); the TMEM panel
// kernel otherwise (a block update touches only G of the SMs, no global all-reduce per
// update).  ASY_DENSE_KERNEL=panel|slab overrides (tests, measurements).
static bool use_slab_kernel(const asy_handle* h, const asy_solve_params* sp) {
    const int want = tuning_of(sp).dense_kernel;
    if (want == ASY_KERNEL_DENSE_PANEL) return false;
    if (want == ASY_KERNEL_DENSE_SLAB || want == ASY_KERNEL_DENSE_SLAB_TMEM) return true;
    // (measured: configs[2], 69 KB per SM per update: slab 3.74 TB/s vs panel 3.22; configs[1],
    // 17 KB: panel 4.4 vs slab 1.8)
    const double per_sm = 8.0 * (double)h->B * (double)h->m / (double)std::max(1, h->sms);
    return per_sm >= 64.0 * 1024.0;
}

#ifndef ASY_SPARSE_DELAY_DIV
#define ASY_SPARSE_DELAY_DIV 4  // auto delay of the CSC kernel: N / this (R25)
#endif
#ifndef ASY_SPARSE_LPC
#define ASY_SPARSE_LPC 2  // lanes per column of the CSC kernel (16 block updates in flight per warp)
#endif
static int sparse_async_launch(asy_handle* h, const asy_solve_params* sp, int64_t sweeps, int64_t delay,
                               float* ms) {
    constexpr int LPC = ASY_SPARSE_LPC;
    void (*kern)(SparseAsyncParams) =
        h->S.loss == LOSS_LS ? sparse_async_kernel<LOSS_LS, LPC> : sparse_async_kernel<LOSS_LOGISTIC, LPC>;
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)kern, kSparseThreads, 0));
    int grid = std::max(1, occ) * h->sms;
    if (sp->workers > 0) grid = std::min(grid, (int)sp->workers);
    // batch size: 32 / LPC updates per warp, at most delay + 1 (a batch never waits for itself)
    const int BS = (int)std::min<int64_t>(32 / LPC, delay + 1);
    const int64_t NB = (h->n + BS - 1) / BS;
    // D1 window counters (sparse_async.cuh): W <= ceil((delay + 2) / BS) - 1 batches per window
    // (the windows a batch waits for end before it); S > (delay + 2) / W + 2 slots (a window is
    // reused only after it completed: delay + 2 sequences span at most delay + 2 batches)
    // (and W <= a sixteenth of the batches the delay spans: the window granularity then costs
    // little of the allowed delay)
    const int64_t wmax = std::max<int64_t>(1, std::min<int64_t>((delay + 2 + BS - 1) / BS - 1, (delay / BS) / 16));
    int lgW = 0;
    while (lgW < 6 && ((int64_t)2 << lgW) <= wmax) ++lgW;
    const int64_t slots = next_pow2(std::max<int64_t>(256, ((delay + 2) >> lgW) + 8));
    int lgS = 0;
    while (((int64_t)1 << lgS) < slots) ++lgS;
    TRY(dev_alloc(h, h->done, sizeof(unsigned) * slots));
    TRY(dev_alloc(h, h->ver, sizeof(unsigned) * h->n));
    TRY(dev_alloc(h, h->rs, sizeof(double) * 2 * h->m));  // [r_i, aux_i] pairs for the launch
    TRY(dev_alloc(h, h->dobs, sizeof(unsigned)));
    SparseAsyncParams P{};
    P.colptr = P_<int64_t>(h->colptr); P.rowidx = P_<int32_t>(h->rowidx); P.vals = P_<double>(h->vals);
    P.m = h->m; P.n = h->n; P.r = P_<double>(h->rs); P.x = P_<double>(h->x);
    P.tau = P_<double>(h->tau); P.S = h->S; P.gamma = sp->gamma; P.sched = sp->schedule; P.seed = sp->seed;
    P.epoch0 = h->epochs; P.T = sweeps * NB; P.NB = NB; P.BS = BS; P.delay = delay;
    P.counter = P_<unsigned long long>(h->counter);
    P.ver = P_<unsigned>(h->ver); P.wcnt = P_<unsigned>(h->done); P.lgW = lgW; P.lgS = lgS;
    P.measure_delay = tuning_of(sp).measure_delay != 0;
    P.use_ver = !(sp->schedule == ASY_SCHED_CYCLIC && delay < h->n);  // D4 implied by D1 (sparse_async.cuh)
    P.dobs = P_<unsigned>(h->dobs);
    h->last_kernel = ASY_KERNEL_SPARSE;
    h->last_delay = (int)delay;
    sparse_async_init<<<grid_for(std::max<int64_t>(slots, h->n), 256, 8 * h->sms), 256, 0, h->stream>>>(P);
    CKL();
    void* args[] = {&P};
    CK(cudaEventRecord(h->ev[0], h->stream));
    sparse_pair_pack<<<grid_for(h->m, 256, 4 * h->sms), 256, 0, h->stream>>>(P_<double>(h->r), P_<double>(h->b),
                                                                             P_<double>(h->rs), h->m);
    CKL();
    CK(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kSparseThreads), args, 0, h->stream));
    sparse_pair_unpack<<<grid_for(h->m, 256, 4 * h->sms), 256, 0, h->stream>>>(P_<double>(h->rs), P_<double>(h->r), h->m);
    CKL();
    CK(cudaEventRecord(h->ev[1], h->stream));
    CK(cudaEventSynchronize(h->ev[1]));
    CKL();
    CK(cudaEventElapsedTime(ms, h->ev[0], h->ev[1]));
    if (P.measure_delay) {
        unsigned dobs = 0;
        CK(cudaMemcpy(&dobs, h->dobs.p, sizeof(unsigned), cudaMemcpyDeviceToHost));
        h->last_dobs = std::max(h->last_dobs, (int)dobs);
    }
    return ASY_OK;
}

ASY_API int asy_solve(asy_handle* h, const asy_solve_params* sp, asy_solve_stats* st) {
    if (!h) return ASY_ERR_INVALID;
    if (!sp) return h->fail(ASY_ERR_INVALID, "asy_solve: params NULL");
    if (!h->has_problem) return h->fail(ASY_ERR_STATE, "asy_solve before asy_set_problem");
    if (!(sp->gamma > 0 && sp->gamma <= 1)) return h->fail(ASY_ERR_INVALID, "gamma must be in (0, 1]");
    if (sp->sweeps < 0) return h->fail(ASY_ERR_INVALID, "sweeps < 0");
    if (sp->mode != ASY_MODE_ASYNC && sp->mode != ASY_MODE_SYNC_JACOBI) return h->fail(ASY_ERR_INVALID, "bad mode");
    if (sp->schedule != ASY_SCHED_CYCLIC && sp->schedule != ASY_SCHED_RANDOM)
        return h->fail(ASY_ERR_INVALID, "bad schedule");
    if (sp->x_mem != ASY_MEM_HOST && sp->x_mem != ASY_MEM_DEVICE) return h->fail(ASY_ERR_INVALID, "bad x_mem");
    if (sp->panel_rows < 0 || (sp->panel_rows % 32) || sp->panel_rows > 256)
        return h->fail(ASY_ERR_INVALID, "panel_rows must be a multiple of 32 in [0, 256]");
    if (sp->stages < 0 || sp->stages > 16) return h->fail(ASY_ERR_INVALID, "stages must be in [0,16]");
    if (sp->tuning) {
        const asy_tuning& t = *sp->tuning;
        if ((t.dense_kernel != 0 && t.dense_kernel != ASY_KERNEL_DENSE_PANEL && t.dense_kernel != ASY_KERNEL_DENSE_SLAB &&
             t.dense_kernel != ASY_KERNEL_DENSE_SLAB_TMEM) ||
            (t.panel_park != 0 && t.panel_park != 2) || t.slab_hold < 0 || t.slab_hold > 2 || t.slab_chunk_rows < 0 ||
            t.slab_chunk_rows > 256 || t.slab_ring < 0 || t.slab_ring > 16 || t.measure_delay < 0 ||
            t.measure_delay > 1)
            return h->fail(ASY_ERR_INVALID, "bad asy_tuning field");
    }
    CK(cudaSetDevice(h->device));
    asy_solve_stats stats{};
    h->last_dobs = -1;
    CK(cudaEventRecord(h->ev[2], h->stream));
    if (sp->reset) TRY(reset_state(h, sp->x0, sp->x_mem));
    int64_t delay = sp->max_delay;
    if (delay < 0) delay = std::max<int64_t>(1, h->nblk / (h->kind == ASY_CSC ? ASY_SPARSE_DELAY_DIV : 8));
    delay = std::min<int64_t>(delay, 1 << 22);
    double kernel_ms = 0;
    int64_t launches = sp->reset ? 2 : 0;
    for (int64_t done = 0; done < sp->sweeps;) {
        const int64_t chunk = sp->f_hist ? 1 : sp->sweeps;
        if (sp->mode == ASY_MODE_SYNC_JACOBI) {
            cudaEventRecord(h->ev[0], h->stream);
            for (int64_t s = 0; s < chunk; ++s) TRY(jacobi_sweep(h, sp->gamma));
            h->last_kernel = ASY_KERNEL_JACOBI;
            h->last_delay = -1;
            cudaEventRecord(h->ev[1], h->stream);
            CK(cudaEventSynchronize(h->ev[1]));
            float ms = 0;
            cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
            kernel_ms += ms;
            launches += chunk * (h->kind == ASY_DENSE_COLMAJOR ? 4 : 3);
        } else {
            float ms = 0;
            if (h->kind == ASY_DENSE_COLMAJOR) {
                bool slab = use_slab_kernel(h, sp), too_tall = false;
                if (!slab) {
                    const int rc = dense_async_launch(h, sp, chunk, delay, &ms, &too_tall);
                    if (rc != ASY_OK && !too_tall) return rc;
                    slab = too_tall;
                }
                if (slab) TRY(dense_slab_launch(h, sp, chunk, delay, &ms));
            }
            else TRY(sparse_async_launch(h, sp, chunk, delay, &ms));
            kernel_ms += ms;
            launches += 2;
        }
        h->epochs += chunk;
        stats.block_updates += chunk * (sp->mode == ASY_MODE_SYNC_JACOBI ? h->nblk : h->nblk);
        if (sp->f_hist) {
            double v[6];
            TRY(reduce_objective(h, P_<double>(h->r), P_<double>(h->x), nullptr, v));
            sp->f_hist[done] = objective_from(h, v, nullptr);
            launches += 2;
        }
        done += chunk;
    }
    {
        double v[6];
        TRY(reduce_objective(h, P_<double>(h->r), P_<double>(h->x), nullptr, v));
        stats.objective = objective_from(h, v, nullptr);
        launches += 2;
    }
    if (sp->x_out)
        CK(cudaMemcpyAsync(sp->x_out, h->x.p, sizeof(double) * h->n,
                           sp->x_mem == ASY_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaEventRecord(h->ev[3], h->stream));
    CK(cudaEventSynchronize(h->ev[3]));
    float tot = 0;
    cudaEventElapsedTime(&tot, h->ev[2], h->ev[3]);
    stats.kernel_ms = kernel_ms;
    stats.total_ms = tot;
    stats.launches = launches;
    stats.epochs = h->epochs;
    stats.kernel = h->last_kernel;
    stats.delay = h->last_delay;
    stats.delay_observed = h->last_dobs;
    if (st) *st = stats;
    return ASY_OK;
}

ASY_API int asy_stationarity(asy_handle* h, const double* x, int32_t x_mem, asy_stationarity_out* out) {
    if (!h) return ASY_ERR_INVALID;
    if (!out) return h->fail(ASY_ERR_INVALID, "out is NULL");
    if (!h->has_problem) return h->fail(ASY_ERR_STATE, "no problem set");
    if (x && x_mem != ASY_MEM_HOST && x_mem != ASY_MEM_DEVICE) return h->fail(ASY_ERR_INVALID, "bad x_mem");
    CK(cudaSetDevice(h->device));
    double* xs = P_<double>(h->xs);
    CK(cudaMemcpyAsync(xs, x ? x : h->x.p, sizeof(double) * h->n,
                       (x && x_mem == ASY_MEM_HOST) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
    // fresh residual, weights, gradient + per-coordinate M_F / merit
    TRY(gemvN(h, xs, h->loss == ASY_LOSS_LS ? COMBINE_FRESH_LS : COMBINE_FRESH_ZERO, P_<double>(h->rs)));
    loss_weights_kernel<<<grid_for(h->m, 256, 4 * h->sms), 256, 0, h->stream>>>(h->S, P_<double>(h->rs),
                                                                                  P_<double>(h->b), P_<double>(h->w), h->m);
    CKL();
    TRY(gemvT(h, P_<double>(h->w), GT_STATIONARITY, xs, 0.0, nullptr, P_<double>(h->mf), P_<double>(h->mer)));
    double v[6];
    TRY(reduce_objective(h, P_<double>(h->rs), xs, P_<double>(h->mf), v));
    out->objective = objective_from(h, v, &out->smooth);
    out->mf_norm2 = sqrt(v[4]);
    out->mf_norminf = v[5];
    max_partial_kernel<<<kRedGrid, kRedThreads, 0, h->stream>>>(P_<double>(h->mer), h->n, P_<double>(h->red_part));
    CKL();
    reduce_final_kernel<<<1, 32, 0, h->stream>>>(P_<double>(h->red_part), kRedGrid, 0x3F, P_<double>(h->red_out));
    CKL();
    double mx[6];
    CK(cudaMemcpyAsync(mx, h->red_out.p, sizeof mx, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    out->merit_inf = mx[0];
    return ASY_OK;
}

ASY_API int asy_get_x(asy_handle* h, double* x, int32_t x_mem) {
    if (!h) return ASY_ERR_INVALID;
    if (!x) return h->fail(ASY_ERR_INVALID, "x is NULL");
    if (!h->has_problem) return h->fail(ASY_ERR_STATE, "no problem set");
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpyAsync(x, h->x.p, sizeof(double) * h->n,
                       x_mem == ASY_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return ASY_OK;
}

ASY_API int asy_get_residual(asy_handle* h, double* r, int32_t r_mem) {
    if (!h) return ASY_ERR_INVALID;
    if (!r) return h->fail(ASY_ERR_INVALID, "r is NULL");
    if (r_mem != ASY_MEM_HOST && r_mem != ASY_MEM_DEVICE) return h->fail(ASY_ERR_INVALID, "bad r_mem");
    if (!h->has_problem) return h->fail(ASY_ERR_STATE, "no problem set");
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpyAsync(r, h->r.p, sizeof(double) * h->m,
                       r_mem == ASY_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return ASY_OK;
}

ASY_API int asy_objective(asy_handle* h, double* F) {
    if (!h) return ASY_ERR_INVALID;
    if (!F) return h->fail(ASY_ERR_INVALID, "F is NULL");
    if (!h->has_problem) return h->fail(ASY_ERR_STATE, "no problem set");
    CK(cudaSetDevice(h->device));
    double v[6];
    TRY(reduce_objective(h, P_<double>(h->r), P_<double>(h->x), nullptr, v));
    *F = objective_from(h, v, nullptr);
    return ASY_OK;
}

ASY_API int asy_schedule_device(asy_handle* h, int32_t schedule, uint64_t seed, int64_t nblocks, int64_t k0,
                                int64_t count, int64_t* out) {
    if (!h) return ASY_ERR_INVALID;
    if (!out || nblocks < 1 || k0 < 0 || count < 0 ||
        (schedule != ASY_SCHED_CYCLIC && schedule != ASY_SCHED_RANDOM))
        return h->fail(ASY_ERR_INVALID, "asy_schedule_device: bad arguments");
    CK(cudaSetDevice(h->device));
    Dev buf;
    TRY(dev_alloc(h, buf, sizeof(int64_t) * std::max<int64_t>(1, count)));
    schedule_kernel<<<grid_for(count, 256, 8 * h->sms), 256, 0, h->stream>>>(schedule, seed, nblocks, k0, count,
                                                                            P_<int64_t>(buf));
    CKL();
    CK(cudaMemcpyAsync(out, buf.p, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    dev_free(buf);
    return ASY_OK;
}

}  // extern "C"
