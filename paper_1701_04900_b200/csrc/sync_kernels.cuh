// sync_kernels.cuh -- deterministic kernels: the synchronous Jacobi sweep
// (two hand-written GEMVs: g = A^T w, then r += A dx), fresh residuals, and
// the objective / stationarity reductions.  Every reduction has a fixed
// order (fixed lane->element map, fixed shuffle tree, fixed-grid two-stage
// sums), so results are bit-reproducible run to run.
#pragma once
#include "common.cuh"

namespace asy {

enum { GT_JACOBI = 0, GT_STATIONARITY = 1 };

// w_j = phi'(r_j)
__global__ void loss_weights_kernel(Scalars S, const double* __restrict__ r,
                                    const double* __restrict__ aux, double* __restrict__ w, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        w[i] = loss_prime(S, r[i], aux[i]);
}

// Per-coordinate epilogue of a computed partial gradient gs = (A^T w)_j.
//   GT_JACOBI:        x_j <- x_j + gamma (hat x_j - x_j), dx_j = new - old   (S.4)
//   GT_STATIONARITY:  mf_j = x_j - argmin(unit metric) (Eq. 5), mer_j = |hat x_j - x_j| (Sec. 4.3)
__device__ __forceinline__ void coord_epilogue(const Scalars& S, int mode, double gs, int64_t j,
                                               double* x, const double* tau, double gamma,
                                               double* dx, double* mf, double* mer) {
    const double y = x[j];
    if (mode == GT_JACOBI) {
        const double xh = best_response(S, gs, y, tau[j], j);
        const double xn = y + gamma * (xh - y);
        x[j] = xn;
        dx[j] = xn - y;
    } else {
        double g = gs - S.c2 * y;
        if (S.reg != REG_L1) g -= S.lam * grad_h_minus(S, y);
        const double yu = coord_argmin(g, y, 1.0, S.lam_eff, box_lo(S, j), box_hi(S, j));
        mf[j] = y - yu;
        const double xh = coord_argmin(g, y, tau[j], S.lam_eff, box_lo(S, j), box_hi(S, j));
        mer[j] = fabs(xh - y);
    }
}

// Dense GEMV-T (+ epilogue): one warp per column, lane l owns rows {2l,2l+1} + 64i.
__global__ void dense_gemvT_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n,
                                   const double* __restrict__ w, Scalars S, int mode, double* x,
                                   const double* __restrict__ tau, double gamma, double* dx,
                                   double* mf, double* mer) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
        const double* col = A + j * lda;
        double acc0 = 0.0, acc1 = 0.0;
        int64_t i = 2 * lane;
        for (; i + 65 < m; i += 128) {
            const double2 a0 = __ldg(reinterpret_cast<const double2*>(col + i));
            const double2 a1 = __ldg(reinterpret_cast<const double2*>(col + i + 64));
            const double2 w0 = __ldg(reinterpret_cast<const double2*>(w + i));
            const double2 w1 = __ldg(reinterpret_cast<const double2*>(w + i + 64));
            acc0 = fma(a0.x, w0.x, acc0); acc0 = fma(a0.y, w0.y, acc0);
            acc1 = fma(a1.x, w1.x, acc1); acc1 = fma(a1.y, w1.y, acc1);
        }
        for (; i < m; i += 64) {
            acc0 = fma(col[i], w[i], acc0);
            if (i + 1 < m) acc0 = fma(col[i + 1], w[i + 1], acc0);
        }
        const double g = warp_sum(acc0 + acc1);
        if (lane == 0) coord_epilogue(S, mode, g, j, x, tau, gamma, dx, mf, mer);
    }
}

// Dense GEMV-N, split over column chunks: part[c][i] = sum_{j in chunk c, v_j != 0} A_ij v_j.
__global__ void dense_gemvN_partial_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                           int64_t n, const double* __restrict__ v, int64_t cpc,
                                           double* __restrict__ part) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t c = blockIdx.y;
    const int64_t j0 = c * cpc, j1 = (j0 + cpc) < n ? (j0 + cpc) : n;
    if (i >= m) return;
    double acc = 0.0;
    int64_t j = j0;
    for (; j + 4 <= j1; j += 4) {
        const double d0 = __ldg(v + j), d1 = __ldg(v + j + 1), d2 = __ldg(v + j + 2), d3 = __ldg(v + j + 3);
        if (d0 == 0.0 && d1 == 0.0 && d2 == 0.0 && d3 == 0.0) continue;
        const double* a = A + j * lda + i;
        const double a0 = d0 != 0.0 ? __ldg(a) : 0.0;
        const double a1 = d1 != 0.0 ? __ldg(a + lda) : 0.0;
        const double a2 = d2 != 0.0 ? __ldg(a + 2 * lda) : 0.0;
        const double a3 = d3 != 0.0 ? __ldg(a + 3 * lda) : 0.0;
        if (d0 != 0.0) acc = fma(a0, d0, acc);
        if (d1 != 0.0) acc = fma(a1, d1, acc);
        if (d2 != 0.0) acc = fma(a2, d2, acc);
        if (d3 != 0.0) acc = fma(a3, d3, acc);
    }
    for (; j < j1; ++j) {
        const double d = __ldg(v + j);
        if (d != 0.0) acc = fma(__ldg(A + j * lda + i), d, acc);
    }
    part[c * m + i] = acc;
}

// out_i = base_i + sum_c part[c][i] (fixed order).  base: r (add) or -b / 0 (fresh).
enum { COMBINE_ADD = 0, COMBINE_FRESH_LS = 1, COMBINE_FRESH_ZERO = 2 };
__global__ void combine_kernel(const double* __restrict__ part, int64_t nchunks, int64_t m,
                               int mode, const double* __restrict__ aux, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t c = 0; c < nchunks; ++c) s += part[c * m + i];
        if (mode == COMBINE_ADD) out[i] = out[i] + s;
        else if (mode == COMBINE_FRESH_LS) out[i] = s - aux[i];
        else out[i] = s;
    }
}

// Sparse GEMV-T (+ epilogue) on CSC: 8 lanes per column, lane g owns entries start+g+8i.
__global__ void csc_gemvT_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                                 const double* __restrict__ vals, int64_t n,
                                 const double* __restrict__ w, Scalars S, int mode, double* x,
                                 const double* __restrict__ tau, double gamma, double* dx,
                                 double* mf, double* mer) {
    const int lane = threadIdx.x & 31, gl = lane & 7;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x >> 3);
    const int64_t g0 = blockIdx.x * (int64_t)(blockDim.x >> 3) + (threadIdx.x >> 3);
    const int64_t iters = (n + groups - 1) / groups;
    for (int64_t it = 0; it < iters; ++it) {   // uniform trip count keeps full-warp shuffles legal
        const int64_t j = g0 + it * groups;
        double acc = 0.0;
        if (j < n) {
            const int64_t s = colptr[j], e = colptr[j + 1];
            for (int64_t q = s + gl; q < e; q += 8) acc = fma(vals[q], w[rowidx[q]], acc);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (j < n && gl == 0) coord_epilogue(S, mode, acc, j, x, tau, gamma, dx, mf, mer);
    }
}

// Sparse GEMV-N on CSR: 8 lanes per row.  out_i = base_i + sum_{q in row i} val_q v_{col_q}.
__global__ void csr_gemvN_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                                 const double* __restrict__ vals, int64_t m,
                                 const double* __restrict__ v, int mode,
                                 const double* __restrict__ aux, double* out) {
    const int lane = threadIdx.x & 31, gl = lane & 7;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x >> 3);
    const int64_t g0 = blockIdx.x * (int64_t)(blockDim.x >> 3) + (threadIdx.x >> 3);
    const int64_t iters = (m + groups - 1) / groups;
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t i = g0 + it * groups;
        double acc = 0.0;
        if (i < m) {
            const int64_t s = rowptr[i], e = rowptr[i + 1];
            for (int64_t q = s + gl; q < e; q += 8) acc = fma(vals[q], v[colidx[q]], acc);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (i < m && gl == 0) {
            if (mode == COMBINE_ADD) out[i] = out[i] + acc;
            else if (mode == COMBINE_FRESH_LS) out[i] = acc - aux[i];
            else out[i] = acc;
        }
    }
}

// ---------------------------------------------------------------------------
// deterministic reductions: fixed grid kRedGrid x 256 threads, then 1 CTA.
// ---------------------------------------------------------------------------
constexpr int kRedGrid = 256;
constexpr int kRedThreads = 256;
constexpr int kRedVals = 6;

__device__ __forceinline__ void block_reduce_store(double (&v)[kRedVals], const bool (&is_max)[kRedVals],
                                                   double* out) {
    __shared__ double sh[kRedThreads / 32][kRedVals];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kRedVals; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double t = __shfl_xor_sync(0xffffffffu, v[q], o);
            v[q] = is_max[q] ? fmax(v[q], t) : v[q] + t;
        }
    }
    if (lane == 0)
        for (int q = 0; q < kRedVals; ++q) sh[warp][q] = v[q];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < kRedVals; ++q) {
            double a = sh[0][q];
            for (int w = 1; w < kRedThreads / 32; ++w) a = is_max[q] ? fmax(a, sh[w][q]) : a + sh[w][q];
            out[q] = a;
        }
    }
}

// partial[cta][0..5] = { sum phi(r), sum x^2, sum h(x), #out-of-box coordinates, sum mf^2,
// max |mf| } (mf = M_F(x) of Eq. 5, only when the stationarity call passes it; the Sec. 4.3
// merit is reduced by max_partial_kernel from its own per-coordinate array)
__global__ void objective_partial_kernel(Scalars S, const double* __restrict__ r,
                                         const double* __restrict__ aux, int64_t m,
                                         const double* __restrict__ x, int64_t n,
                                         const double* __restrict__ mf, double* partial) {
    double v[kRedVals] = {0, 0, 0, 0, 0, 0};
    const bool is_max[kRedVals] = {false, false, false, false, false, true};
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < m; i += nth) v[0] += loss_value(S, r[i], aux[i]);
    for (int64_t j = tid; j < n; j += nth) {
        const double xj = x[j];
        v[1] += xj * xj;
        v[2] += reg_value(S, xj);
        if (xj < box_lo(S, j) || xj > box_hi(S, j)) v[3] += 1.0;
        if (mf) { v[4] += mf[j] * mf[j]; v[5] = fmax(v[5], fabs(mf[j])); }
    }
    block_reduce_store(v, is_max, partial + blockIdx.x * kRedVals);
}

// max of an array (merit) -- fixed grid partial maxima
__global__ void max_partial_kernel(const double* __restrict__ a, int64_t n, double* partial) {
    double v[kRedVals] = {0, 0, 0, 0, 0, 0};
    const bool is_max[kRedVals] = {true, true, true, true, true, true};
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        v[0] = fmax(v[0], a[j]);
    block_reduce_store(v, is_max, partial + blockIdx.x * kRedVals);
}

// final: out[q] = fixed-order combination of partial[0..kRedGrid)[q]
__global__ void reduce_final_kernel(const double* __restrict__ partial, int nparts, int max_mask,
                                    double* out) {
    const int q = threadIdx.x;
    if (q >= kRedVals) return;
    const bool mx = (max_mask >> q) & 1;
    double a = partial[q];
    for (int c = 1; c < nparts; ++c) a = mx ? fmax(a, partial[c * kRedVals + q]) : a + partial[c * kRedVals + q];
    out[q] = a;
}

// x0 = projection of 0 onto the box X (Algorithm 1 initialisation, x^0 in X [PAPER.md:250])
__global__ void project_zero_kernel(Scalars S, double* x, int64_t n) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        x[j] = fmin(fmax(0.0, box_lo(S, j)), box_hi(S, j));
}

// x <- value / copy helpers
__global__ void fill_kernel(double* a, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

__global__ void fresh_residual_base_kernel(double* r, const double* __restrict__ aux, int64_t m, int ls) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = ls ? -aux[i] : 0.0;
}

// validation: count tau <= 0 / non-finite, lo > hi
__global__ void validate_kernel(const double* tau, const double* lo, const double* hi, int64_t n,
                                unsigned long long* bad) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double t = tau[j];
        bool b = !(t > 0.0) || isinf(t);
        if (lo && hi && lo[j] > hi[j]) b = true;
        if (b) atomicAdd(bad, 1ull);
    }
}

__global__ void schedule_kernel(int sched, uint64_t seed, int64_t nblocks, int64_t k0, int64_t count,
                                int64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = schedule_block(sched, seed, nblocks, k0 + i);
}

// CSC -> CSR helpers
__global__ void expand_colids_kernel(const int64_t* __restrict__ colptr, int64_t n, int32_t* colid) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) colid[q] = (int32_t)j;
}
__global__ void iota_kernel(int32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}
__global__ void row_count_kernel(const int32_t* __restrict__ rowidx, int64_t nnz, int64_t m,
                                 int64_t* counts, unsigned long long* bad) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = rowidx[q];
        if (r < 0 || r >= m) atomicAdd(bad, 1ull);
        else atomicAdd(reinterpret_cast<unsigned long long*>(counts + r), 1ull);
    }
}
__global__ void csr_gather_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ colid,
                                  const double* __restrict__ vals, int64_t nnz, int32_t* ccol, double* cval) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = perm[i];
        ccol[i] = colid[p];
        cval[i] = vals[p];
    }
}

}  // namespace asy
