// Stage-level anchor mapping from a given set of eight channels (sm_100a).
//
// The engine never materialises channels (det_sat.cuh goes straight from labels to the
// residual field).  These two kernels serve the reference's stage API on an arbitrary
// IntegralImageSet, with the reference's float64 op order (explicit _rn intrinsics, no FMA
// contraction), so the result is a function of the channels alone:
//   k_map_grid   mapping_grid (displacement.py:102-131), optionally minus a base grid
//                (residual_field, displacement.py:198-206);
//   k_map_points mapping_point (displacement.py:150-170): straight channels sampled on the
//                (n+1)^2 corner lattice (_corner_lattice, :77-92), tilted channels between
//                pixel centres (_sample_lattice, :134-147).
// Channel layout: ch[c][j][i], c = alpha, beta, gamma, delta, alpha_t, beta_t, gamma_t, delta_t.
#pragma once
#include "det_common.cuh"

namespace det {

// ext[j][i] of the corner lattice: 0 on the virtual first row/column, alpha[j-1][i-1] otherwise
__device__ __forceinline__ double lat_ext(const double* __restrict__ alpha, int n, int j, int i) {
    return (i == 0 || j == 0) ? 0.0 : alpha[(size_t)(j - 1) * n + (i - 1)];
}

// anchor coordinates of the pixel centre / point (x, y) (displacement.py:35-74), same op order
struct Anch {
    double q1x, q1y, q2x, q2y, q3x, q3y, q4x, q4y;
};
__device__ __forceinline__ Anch anchors_at(double x, double y) {
    Anch a;
    if (y < x) {
        a.q1x = 1.0; a.q1y = __dsub_rn(__dadd_rn(1.0, y), x);
        a.q3x = __dsub_rn(x, y); a.q3y = 0.0;
    } else {
        a.q1x = __dadd_rn(__dsub_rn(1.0, y), x); a.q1y = 1.0;
        a.q3x = 0.0; a.q3y = __dsub_rn(y, x);
    }
    const double s = __dadd_rn(x, y);
    if (s < 1.0) {
        a.q2x = s; a.q2y = 0.0;
        a.q4x = 0.0; a.q4y = s;
    } else {
        a.q2x = 1.0; a.q2y = __dsub_rn(s, 1.0);
        a.q4x = __dsub_rn(s, 1.0); a.q4y = 1.0;
    }
    return a;
}

// mapping_grid: one thread per pixel centre.  base == nullptr -> t(d); else t(d) - base.
__global__ void k_map_grid(const double* __restrict__ ch, double total, int n, const double* __restrict__ base,
                           double* __restrict__ out) {
    const size_t nn = (size_t)n * n;
    const double* alpha = ch;
    const double inv = __ddiv_rn(1.0, __dmul_rn(2.0, total));
    for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < nn; p += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(p / n), i = (int)(p - (size_t)j * n);
        // a = 0.25 * (ext[:-1,:-1] + ext[:-1,1:] + ext[1:,:-1] + ext[1:,1:])
        const double e00 = lat_ext(alpha, n, j, i), e01 = lat_ext(alpha, n, j, i + 1);
        const double e10 = lat_ext(alpha, n, j + 1, i), e11 = lat_ext(alpha, n, j + 1, i + 1);
        const double a = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(e00, e01), e10), e11));
        const double col_avg = __dmul_rn(0.5, __dadd_rn(lat_ext(alpha, n, n, i), lat_ext(alpha, n, n, i + 1)));
        const double row_avg = __dmul_rn(0.5, __dadd_rn(lat_ext(alpha, n, j, n), lat_ext(alpha, n, j + 1, n)));
        const double b = __dsub_rn(col_avg, a);
        const double d = __dsub_rn(row_avg, a);
        const double g = __dadd_rn(__dsub_rn(__dsub_rn(total, col_avg), row_avg), a);
        const double at = ch[4 * nn + p], bt = ch[5 * nn + p], gt = ch[6 * nn + p], dt = ch[7 * nn + p];
        // c = (arange(n) + 0.5) / n
        const double x = __ddiv_rn((double)i + 0.5, (double)n), y = __ddiv_rn((double)j + 0.5, (double)n);
        const Anch q = anchors_at(x, y);
        double tx = __dmul_rn(a, q.q1x);
        tx = __dadd_rn(tx, __dmul_rn(b, q.q2x));
        tx = __dadd_rn(tx, __dmul_rn(g, q.q3x));
        tx = __dadd_rn(tx, __dmul_rn(d, q.q4x));
        tx = __dadd_rn(tx, __dmul_rn(at, x));
        tx = __dadd_rn(tx, bt);
        tx = __dadd_rn(tx, __dmul_rn(gt, x));
        tx = __dmul_rn(tx, inv);
        double ty = __dmul_rn(a, q.q1y);
        ty = __dadd_rn(ty, __dmul_rn(b, q.q2y));
        ty = __dadd_rn(ty, __dmul_rn(g, q.q3y));
        ty = __dadd_rn(ty, __dmul_rn(d, q.q4y));
        ty = __dadd_rn(ty, at);
        ty = __dadd_rn(ty, __dmul_rn(bt, y));
        ty = __dadd_rn(ty, __dmul_rn(dt, y));
        ty = __dmul_rn(ty, inv);
        if (base) {
            tx = __dsub_rn(tx, base[2 * p]);
            ty = __dsub_rn(ty, base[2 * p + 1]);
        }
        out[2 * p] = tx;
        out[2 * p + 1] = ty;
    }
}

// _sample_lattice (displacement.py:134-147) of node values given by `val(j, i)` on an
// m x m node grid
template <typename F>
__device__ __forceinline__ double sample_lattice(F val, int m, double gx, double gy) {
    const double hi = (double)(m - 2);
    const double bx = fmin(fmax(floor(gx), 0.0), hi), by = fmin(fmax(floor(gy), 0.0), hi);
    const int i0 = (int)bx, j0 = (int)by;
    const double fx = fmin(fmax(__dsub_rn(gx, (double)i0), 0.0), 1.0);
    const double fy = fmin(fmax(__dsub_rn(gy, (double)j0), 0.0), 1.0);
    const double gxm = __dsub_rn(1.0, fx), gym = __dsub_rn(1.0, fy);
    double s = __dmul_rn(__dmul_rn(val(j0, i0), gxm), gym);
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(val(j0, i0 + 1), fx), gym));
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(val(j0 + 1, i0), gxm), fy));
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(val(j0 + 1, i0 + 1), fx), fy));
    return s;
}

// mapping_point: one thread per query point (x, y) in [0, 1]^2.
__global__ void k_map_points(const double* __restrict__ ch, double total, int n, const double2* __restrict__ pts,
                             int np, double2* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= np) return;
    const size_t nn = (size_t)n * n;
    const double* alpha = ch;
    const double x = pts[t].x, y = pts[t].y;
    const double nd = (double)n;
    const double gx = __dmul_rn(x, nd), gy = __dmul_rn(y, nd);
    // straight channels on the corner lattice (_corner_lattice): ext, beta_ext = col_full - ext,
    // gamma_ext = total - col_full - row_full + ext, delta_ext = row_full - ext
    auto ext = [&](int j, int i) { return lat_ext(alpha, n, j, i); };
    double w[8];
    w[0] = sample_lattice(ext, n + 1, gx, gy);
    w[1] = sample_lattice([&](int j, int i) { return __dsub_rn(ext(n, i), ext(j, i)); }, n + 1, gx, gy);
    w[2] = sample_lattice(
        [&](int j, int i) { return __dadd_rn(__dsub_rn(__dsub_rn(total, ext(n, i)), ext(j, n)), ext(j, i)); }, n + 1,
        gx, gy);
    w[3] = sample_lattice([&](int j, int i) { return __dsub_rn(ext(j, n), ext(j, i)); }, n + 1, gx, gy);
    const double tx = __dsub_rn(gx, 0.5), ty = __dsub_rn(gy, 0.5);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const double* tc = ch + (4 + c) * nn;
        w[4 + c] = sample_lattice([&](int j, int i) { return tc[(size_t)j * n + i]; }, n, tx, ty);
    }
    const Anch q = anchors_at(x, y);
    // points q1, q2, q3, q4, e1 = (x, 1), e2 = (1, y), e3 = (x, 0), e4 = (0, y)
    const double px[8] = {q.q1x, q.q2x, q.q3x, q.q4x, x, 1.0, x, 0.0};
    const double py[8] = {q.q1y, q.q2y, q.q3y, q.q4y, 1.0, y, 0.0, y};
    double ax = 0.0, ay = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        ax = __dadd_rn(ax, __dmul_rn(w[c], px[c]));
        ay = __dadd_rn(ay, __dmul_rn(w[c], py[c]));
    }
    const double den = __dmul_rn(2.0, total);
    out[t] = make_double2(__ddiv_rn(ax, den), __ddiv_rn(ay, den));
}

}  // namespace det
