// Straight + 45-degree-tilted integral images -> displacement field (sm_100a).
//
// Replaces integral.py:47-169 (straight_inims / tilted_inims) and
// displacement.py:102-131,198-206 (mapping_grid - base_mapping) with three
// band-parallel kernels that never materialise the eight channels:
//
//   rho(j,i) = m * d(j,i) / C - 1      (residual density; by linearity of every
//                                       channel, u = t(d) - t(const) equals the
//                                       anchor combination of rho's channels / 2m)
//   A(j,i)   = sum_{i'<=i} rho(j,i')   (row prefix, clamped: A(j,i>=n) = row total)
//
// Straight channels come from alpha(j,i) = sum_{j'<=j} A(j',i).  The tilted ones
// come from the rotated-lattice sums R(U,V) = sum_{i'+j'<=U, i'-j'<=V} rho, which
// split into an up-left diagonal prefix UL of A above the row and a down-left one
// DL at/below it:  R(U,V) = UL(j-1,i-1) + DL(j,i)  (U=i+j, V=i-j), and
//   left   beta_t  = R(U,V-1)              = UL(j,i-1)   + DL(j+1,i-1)
//   top    alpha_t = Tu(U-1) - R(U-1,V-1) + rho(j,i),   R(U-1,V-1) = UL(j-1,i-2) + DL(j,i-1)
//   bottom gamma_t = Tv(V) - R(U,V)
//   right  delta_t = C - alpha_t - beta_t - gamma_t
// with Tu/Tv the anti-diagonal / diagonal prefix totals.  This reproduces the
// reference's sector tie rule (integral.py:9-14, oracle tests/oracles.py:30-54).
//
// The texture is cut into bands of H rows (one CTA per band and cartogram):
//   k_sat1  per-band sums of rho along columns, diagonals and anti-diagonals
//           (streamed one row at a time, one barrier per row), x-prefixed once at
//           the band end, plus row totals;
//   k_sat2  band-direction exclusive prefixes / inclusive suffixes (the carries)
//           and image totals -- every value k_sat3 needs, ready to load;
//   k_sat3  per band: load the carries, then one top-down sweep computing A,
//           alpha, UL and the in-band up-right ray URin (DL = DLtot - URin), and
//           the displacement u at every pixel centre (or the 8 channels).
// All accumulation is float64; only the stored field may be float32.
#pragma once
#include "det_common.cuh"

namespace det {

// Residual density of CPT consecutive pixels of row j in the accumulator type A
// (float32 in the float32-field mode, float64 otherwise).
template <int CPT, int SRC, typename A>
__device__ __forceinline__ void load_rho(const Bufs& D, const SatSrc& S, int R, int b, int j, int x0, A (&rho)[CPT]) {
    const int n = D.n;
    if (x0 >= n) {
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = (A)0;
        return;
    }
    if (SRC == SRC_LABELS) {
        const int* lab = D.labels + (size_t)b * D.nn + (size_t)j * n + x0;
        int L[CPT];
        if (CPT == 2) {
            const int2 v = *reinterpret_cast<const int2*>(lab);
            L[0] = v.x; L[1] = v.y;
        } else {
#pragma unroll
            for (int q = 0; q < CPT; q += 4) {
                const int4 v = *reinterpret_cast<const int4*>(lab + q);
                L[q] = v.x; L[q + 1] = v.y; L[q + 2] = v.z; L[q + 3] = v.w;
            }
        }
        if (sizeof(A) == 4) {
            const float* lut = D.lutf + (size_t)b * (R + 1);
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = (A)__ldg(lut + (L[k] < 0 ? R : L[k]));
        } else {
            const double* lut = D.lut + (size_t)b * (R + 1);
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = (A)__ldg(lut + (L[k] < 0 ? R : L[k]));
        }
    } else {
        const double* d = S.d + (size_t)b * D.nn + (size_t)j * n + x0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = (A)__dadd_rn(__dmul_rn(d[k], S.scale), S.offset);
    }
}

template <typename A>
__device__ __forceinline__ A warp_incl_scan_t(A v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const A t = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// In-place inclusive prefix of a[0..len) in shared memory by the whole CTA (float64 carry).
template <typename A>
__device__ void block_prefix_smem(A* a, double* out, int len, double* sm) {
    const int nt = blockDim.x;
    const int per = (len + nt - 1) / nt;
    const int s = min(len, threadIdx.x * per), e = min(len, s + per);
    double loc = 0.0;
    for (int i = s; i < e; ++i) loc += (double)a[i];
    double tot;
    double run = block_excl_scan(loc, sm, &tot);
    for (int i = s; i < e; ++i) {
        run += (double)a[i];
        out[i] = run;
    }
}

// ---------------------------------------------------------------------------------
// Per-band sums, x-prefixed:  CS_b(x) = sum_{j in band, i<=x} rho,
// DG_b(v) = sum_{j in band, i-j<=v} rho (compact index q = v + jb, q in [0, n+H-1)),
// AD_b(w) = sum_{j in band, i+j<=w} rho (compact index q = w - jt).  Outside the
// compact range the prefixes are 0 (below) or the band total (above).  In-band sums
// in A; the x-prefixes and everything downstream in float64.
template <int CPT, int NT, int SRC, typename A>
__global__ void __launch_bounds__(NT) k_sat1(Topo T, Bufs D, SatSrc S, int gate) {
    extern __shared__ unsigned char s_raw1[];  // dg[L] | ad[L] in A
    __shared__ A s_w[3][32];
    __shared__ A s_bd[3][32];
    __shared__ A s_ba[3][32];
    __shared__ double s_red[33];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, L = n + H - 1;
    const int x0 = t * CPT;
    const size_t bb = (size_t)b * D.nb + band;
    A* dg = reinterpret_cast<A*>(s_raw1);
    A* ad = dg + L;
    A cs[CPT], pd[CPT], pa[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) cs[k] = pd[k] = pa[k] = (A)0;

    A rho_n[CPT];
    load_rho<CPT, SRC, A>(D, S, T.R, b, jt, x0, rho_n);
    for (int j = jt; j <= jb; ++j) {
        const int slot = (j - jt) % 3, ps = (j - jt + 2) % 3;
        A rho[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
        if (j < jb) load_rho<CPT, SRC, A>(D, S, T.R, b, j + 1, x0, rho_n);  // prefetch the next row
        A ts = (A)0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) ts += rho[k];
        ts = warp_sum(ts);
        if (lane == 0) s_w[slot][w] = ts;
        __syncthreads();
        A left = __shfl_up_sync(FULL, pd[CPT - 1], 1);
        A right = __shfl_down_sync(FULL, pa[0], 1);
        if (lane == 0) left = (w == 0 || j == jt) ? (A)0 : s_bd[ps][w - 1];
        if (lane == 31) right = (w == nw - 1 || j == jt) ? (A)0 : s_ba[ps][w + 1];
        A nd_[CPT], na_[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            nd_[k] = rho[k] + (k == 0 ? left : pd[k - 1]);
            na_[k] = rho[k] + (k == CPT - 1 ? right : pa[k + 1]);
            cs[k] += rho[k];
        }
        if (t == 0) {
            double s = 0.0;
            for (int q = 0; q < nw; ++q) s += (double)s_w[slot][q];
            D.rt[(size_t)b * n + j] = s;
        }
        if (j < jb) {
            if (x0 <= n - 1 && n - 1 < x0 + CPT) dg[n - 1 - j + jb] = nd_[n - 1 - x0];  // diagonal leaves right edge
            if (x0 == 0) ad[j - jt] = na_[0];                                           // anti-diagonal leaves left edge
        }
        if (lane == 31) s_bd[slot][w] = nd_[CPT - 1];
        if (lane == 0) s_ba[slot][w] = na_[0];
#pragma unroll
        for (int k = 0; k < CPT; ++k) { pd[k] = nd_[k]; pa[k] = na_[k]; }
    }
    // band bottom: remaining diagonals / anti-diagonals end here; column sums -> x-prefix
    double csum = 0.0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        if (x < n) {
            dg[x] = pd[k];
            ad[jb - jt + x] = pa[k];
        }
        csum += x < n ? (double)cs[k] : 0.0;
    }
    double tot;
    double run = block_excl_scan(csum, s_red, &tot);  // (its barriers also publish dg/ad)
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        run += (double)cs[k];
        if (x < n) D.cs[bb * n + x] = run;
    }
    block_prefix_smem<A>(dg, D.dgc + bb * L, L, s_red);
    block_prefix_smem<A>(ad, D.adc + bb * L, L, s_red);
}

// ---------------------------------------------------------------------------------
// float32 path, smem-staged: the band's H x n residual densities are loaded once (all
// label/LUT loads independent -> high memory-level parallelism) into shared memory.
constexpr int LUT_SMEM_MAX = 16384;  // float LUT entries copied to shared memory per CTA

// Copy the cartogram's float LUT (R+1 entries) into shared memory when it fits; returns the
// table to gather from (smem copy or the global array).
__device__ __forceinline__ const float* stage_lut(const Bufs& D, int R, int b, float* s_lut) {
    const float* g = D.lutf + (size_t)b * (R + 1);
    if (R + 1 > LUT_SMEM_MAX) return g;
    for (int i = threadIdx.x; i <= R; i += blockDim.x) s_lut[i] = __ldg(g + i);
    __syncthreads();
    return s_lut;
}

template <int CPT>
__device__ __forceinline__ void stage_rho_band(const Bufs& D, const float* lut, int R, int b, int jt, int H, int x0,
                                               float* rho) {
    const int n = D.n;
    if (x0 >= n) return;
    const int* lab = D.labels + (size_t)b * D.nn + (size_t)jt * n + x0;
    for (int j0 = 0; j0 < H; j0 += 4) {
        int L[4][CPT];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (j0 + q >= H) continue;
#pragma unroll
            for (int k = 0; k < CPT; k += 2) {
                const int2 v = *reinterpret_cast<const int2*>(lab + (size_t)(j0 + q) * n + k);
                L[q][k] = v.x;
                L[q][k + 1] = v.y;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (j0 + q >= H) continue;
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[(j0 + q) * n + x0 + k] = lut[L[q][k] < 0 ? R : L[q][k]];
        }
    }
}

// k_sat1 for the float32 path: band sums straight from the staged band, no per-row barriers.
template <int CPT, int NT>
__global__ void __launch_bounds__(NT) k_sat1s(Topo T, Bufs D, int gate) {
    extern __shared__ float s_f1[];  // rho[H][n] | dg[L] | ad[L] | lut[R+1]
    __shared__ double s_red[33];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, L = n + H - 1;
    const int x0 = t * CPT;
    const size_t bb = (size_t)b * D.nb + band;
    float* rho = s_f1;
    float* dg = rho + H * n;
    float* ad = dg + L;
    const float* lut = stage_lut(D, T.R, b, ad + L);
    stage_rho_band<CPT>(D, lut, T.R, b, jt, H, x0, rho);
    __syncthreads();
    for (int jj = w; jj < H; jj += nw) {  // row totals
        float s = 0.f;
        for (int x = lane; x < n; x += 32) s += rho[jj * n + x];
        s = warp_sum(s);
        if (lane == 0) D.rt[(size_t)b * n + jt + jj] = (double)s;
    }
    for (int q = t; q < L; q += blockDim.x) {
        float sd = 0.f, sa = 0.f;
        for (int jj = 0; jj < H; ++jj) {
            const int xd = q - (H - 1) + jj;  // diagonal q = x - j + jb
            const int xa = q - jj;            // anti-diagonal q = x + j - jt
            if (xd >= 0 && xd < n) sd += rho[jj * n + xd];
            if (xa >= 0 && xa < n) sa += rho[jj * n + xa];
        }
        dg[q] = sd;
        ad[q] = sa;
    }
    double cs[CPT], csum = 0.0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        float c = 0.f;
        const int x = x0 + k;
        if (x < n)
            for (int jj = 0; jj < H; ++jj) c += rho[jj * n + x];
        cs[k] = (double)c;
        csum += cs[k];
    }
    double tot;
    double run = block_excl_scan(csum, s_red, &tot);  // (its barriers also publish dg/ad)
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        run += cs[k];
        if (x < n) D.cs[bb * n + x] = run;
    }
    block_prefix_smem<float>(dg, D.dgc + bb * L, L, s_red);
    block_prefix_smem<float>(ad, D.adc + bb * L, L, s_red);
}

// ---------------------------------------------------------------------------------
// Band-direction carries.  Lanes: [0,n) columns x, [n,3n-1) diagonals (idx=v+n-1),
// [3n-1,5n-2) anti-diagonals w.  blockDim = 32*G (G band groups).  The last block
// column computes rowfull (row-total prefix) instead.  Outputs per band b:
//   csX[b][x]   = sum_{b'<b} CS_b'(x)                 (alpha carry)
//   dgXc[b][x]  = sum_{b'<b} DG_b'(x - jt + 1)        (UL carry, x in [0,n))
//   adSc[b][q]  = sum_{b'>=b} AD_b'(jt - 1 + q)        (DLtot window, q in [0,n+H))
// and totals csT[x] = colfull(x+1), dgT[idx] = Tv(v), adT[w] = Tu(w).
__global__ void k_sat2(Bufs D, int gate) {
    __shared__ double s_g[32][33];
    __shared__ double s_red[33];
    const int b = blockIdx.y + D.b0, t = threadIdx.x, lx = t & 31, g = t >> 5, G = blockDim.x >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, nb = D.nb, L = n + H - 1, M = 2 * n - 1;
    if (blockIdx.x == gridDim.x - 1) {
        // rowfull[J] = sum_{j<J} rt[j]
        const double* rt = D.rt + (size_t)b * n;
        double* rf = D.rowfull + (size_t)b * (n + 1);
        const int per = (n + blockDim.x - 1) / blockDim.x;
        const int a = min(n, t * per), e = min(n, a + per);
        double s = 0.0;
        for (int i = a; i < e; ++i) s += rt[i];
        double tot;
        double run = block_excl_scan(s, s_red, &tot);
        for (int i = a; i < e; ++i) { rf[i] = run; run += rt[i]; }
        if (t == 0) rf[n] = tot;
        return;
    }
    const int lanes = n + 2 * M;
    const int l = blockIdx.x * 32 + lx;
    const bool valid = l < lanes;
    const int type = l < n ? 0 : (l < n + M ? 1 : 2);
    const int idx = type == 0 ? l : (type == 1 ? l - n : l - n - M);
    const int per = (nb + G - 1) / G;
    const int bA = min(nb, g * per), bE = min(nb, bA + per);
    const size_t base = (size_t)b * nb;

    auto val = [&](int band) -> double {
        if (!valid) return 0.0;
        if (type == 0) return D.cs[(base + band) * n + idx];
        int q;
        const double* arr;
        if (type == 1) {
            q = idx - (n - 1) + (band * H + H - 1);  // v + jb
            arr = D.dgc;
        } else {
            q = idx - band * H;                      // w - jt
            arr = D.adc;
        }
        if (q < 0) return 0.0;
        return arr[(base + band) * L + min(q, L - 1)];
    };
    double sum = 0.0;
    for (int band = bA; band < bE; ++band) sum += val(band);
    s_g[g][lx] = sum;
    __syncthreads();
    double before = 0.0, after = 0.0, total = 0.0;
    for (int q = 0; q < G; ++q) {
        const double v = s_g[q][lx];
        total += v;
        if (q < g) before += v;
        if (q > g) after += v;
    }
    if (!valid) return;
    if (type != 2) {
        double run = before;
        for (int band = bA; band < bE; ++band) {
            if (type == 0) {
                D.csX[(base + band) * n + idx] = run;
            } else {
                const int x = idx - n + band * H;  // v + jt - 1, v = idx - (n-1)
                if (x >= 0 && x < n) D.dgXc[(base + band) * n + x] = run;
            }
            run += val(band);
        }
    } else {
        double run = after;
        for (int band = bE - 1; band >= bA; --band) {
            run += val(band);
            const int q = idx - band * H + 1;  // w - (jt - 1)
            if (q >= 0 && q < L + 1) D.adSc[(base + band) * (L + 1) + q] = run;
        }
    }
    if (g == 0) {
        if (type == 0) D.csT[(size_t)b * n + idx] = total;
        else if (type == 1) D.dgT[(size_t)b * M + idx] = total;
        else D.adT[(size_t)b * M + idx] = total;
    }
}

// ---------------------------------------------------------------------------------
// Per band: load the float64 carries, then one top-down sweep.  In-band arithmetic
// in A (float32 when the field is stored as float32), carries rounded to A once.
template <int CPT, int NT, int SRC, typename UT, int OUT, typename A, bool STAGE>
__global__ void __launch_bounds__(NT) k_sat3(Topo T, Bufs D, SatSrc S, int gate) {
    extern __shared__ unsigned char s_raw3[];
    __shared__ A s_w[3][32];
    __shared__ A s_xa[3][32], s_xu1[3][32], s_xu2[3][32], s_xr[3][32];
    const int band = blockIdx.x, b = blockIdx.y + D.b0, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, M = 2 * n - 1;
    const int x0 = t * CPT;
    const size_t bb = (size_t)b * D.nb + band;
    const int WN = n + H;
    A* win_dl = reinterpret_cast<A*>(s_raw3);  // DLtot(w), w in [jt-1, jb+n-1]  -> [w-(jt-1)]
    A* win_tu = win_dl + WN;                   // Tu(w),    w in [jt-1, jb+n-2]  -> [w-(jt-1)]
    A* win_tv = win_dl + 2 * WN;               // Tv(v),    v in [-jb, n-1-jt]   -> [v+jb]
    const double* rowfull = D.rowfull + (size_t)b * (n + 1);
    const double* adT = D.adT + (size_t)b * M;
    const double* dgT = D.dgT + (size_t)b * M;
    const double* csT = D.csT + (size_t)b * n;

    // ---- carries (k_sat2) ----
    for (int q = t; q < WN; q += blockDim.x) {
        win_dl[q] = (jt == 0 && q == 0) ? (A)0 : (A)D.adSc[bb * WN + q];  // DLtot(-1) = 0
        const int wq = jt - 1 + q;
        win_tu[q] = (wq >= 0 && wq < M) ? (A)adT[wq] : (A)0;
        const int iv = q - jb + n - 1;  // Tv index of v = q - jb
        win_tv[q] = (iv >= 0 && iv < M) ? (A)dgT[iv] : (A)0;
    }
    // cc[k]: column-total average cavg(x) = (colfull(x) + colfull(x+1))/2 for the field,
    // colfull(x+1) for the channel dump
    A ul[CPT], al[CPT], cc[CPT], ur[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        const bool in = x < n;
        al[k] = in ? (A)D.csX[bb * n + x] : (A)0;
        ul[k] = in ? (A)D.dgXc[bb * n + x] : (A)0;
        const double cfi = in ? csT[x] : 0.0, cfe = (in && x > 0) ? csT[x - 1] : 0.0;
        cc[k] = (A)(OUT == OUT_CH8 ? cfi : 0.5 * (cfe + cfi));
        ur[k] = (A)0;
    }
    if (lane == 31) {  // boundary values of "row jt-1" = carries
        s_xa[2][w] = al[CPT - 1];
        s_xu1[2][w] = ul[CPT - 1];
        s_xu2[2][w] = ul[CPT - 2];
    }
    if (lane == 0) s_xr[2][w] = (A)0;
    const double rf_top = rowfull[jt];
    const A Cr = (A)rowfull[n];
    const double inv_nd = 1.0 / (double)n;  // exact: n is a power of two
    const A inv_n = (A)inv_nd;
    const A inv2m = (A)(S.outscale != 0.0 ? S.outscale : 0.5 * inv_nd * inv_nd);
    const A xc0 = (A)(((double)x0 + 0.5) * inv_nd);  // pixel-centre x of column x0 (displacement.py:59)
    UT* uf = reinterpret_cast<UT*>(D.uf) + (size_t)b * D.nn * 2;
    constexpr bool STAGED = STAGE && (sizeof(A) == 4 && SRC == SRC_LABELS);
    float* srho = reinterpret_cast<float*>(win_dl + 3 * WN);  // staged band (float path)
    A* s_ex = reinterpret_cast<A*>(srho + (size_t)H * n);      // A(j, x0-1) per (row, thread)
    __shared__ A s_wt[64][33];                                      // warp totals per row (H <= 64)
    A rho_n[CPT];
    if (STAGED) {
        const float* lut = stage_lut(D, T.R, b, reinterpret_cast<float*>(s_ex + (size_t)H * NT));
        stage_rho_band<CPT>(D, lut, T.R, b, jt, H, x0, srho);
        __syncthreads();
        // all H row prefixes up front: the scans are independent across rows (ILP), so the
        // sequential row loop below only carries the vertical/diagonal recurrences
        for (int j0 = 0; j0 < H; j0 += 4) {
            A ts[4], wi[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                ts[q] = (A)0;
                if (j0 + q < H && x0 < n) {
#pragma unroll
                    for (int k = 0; k < CPT; ++k) ts[q] += (A)srho[(j0 + q) * n + x0 + k];
                }
                wi[q] = ts[q];
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const A y = __shfl_up_sync(FULL, wi[q], o);
                    if (lane >= o) wi[q] += y;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (j0 + q >= H) continue;
                if (lane == 31) s_wt[j0 + q][w] = wi[q];
                s_ex[(j0 + q) * NT + t] = wi[q] - ts[q];
            }
        }
        __syncthreads();
        if (t < H) {  // exclusive prefix of the warp totals of row t, stored in place
            A run = (A)0;
            for (int q = 0; q < nw; ++q) {
                const A v = s_wt[t][q];
                s_wt[t][q] = run;
                run += v;
            }
        }
    } else {
        load_rho<CPT, SRC, A>(D, S, T.R, b, jt, x0, rho_n);
    }
    __syncthreads();

    for (int j = jt; j <= jb; ++j) {
        const int slot = (j - jt) % 3, ps = (j - jt + 2) % 3;
        A rho[CPT];
        if (STAGED) {
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = x0 < n ? (A)srho[(j - jt) * n + x0 + k] : (A)0;
        } else {
#pragma unroll
            for (int k = 0; k < CPT; ++k) rho[k] = rho_n[k];
            if (j < jb) load_rho<CPT, SRC, A>(D, S, T.R, b, j + 1, x0, rho_n);  // prefetch the next row
        }
        A loc[CPT];
        A run = (A)0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) { run += rho[k]; loc[k] = run; }
        A excl;  // A(j, x0-1)
        if (STAGED) {
            excl = s_ex[(j - jt) * NT + t] + s_wt[j - jt][w];
            __syncthreads();  // boundary values of the previous row (s_x*) are published
        } else {
            const A tsum = run;
            const A winc = warp_incl_scan_t<A>(tsum);
            if (lane == 31) s_w[slot][w] = winc;
            __syncthreads();
            A off = (A)0;
            for (int q = 0; q < w; ++q) off += s_w[slot][q];
            excl = off + winc - tsum;
        }
        A ap_m1 = __shfl_up_sync(FULL, al[CPT - 1], 1);
        A ul_m1 = __shfl_up_sync(FULL, ul[CPT - 1], 1);
        A ul_m2 = __shfl_up_sync(FULL, ul[CPT - 2], 1);
        A ur_p = __shfl_down_sync(FULL, ur[0], 1);
        if (lane == 0) {
            if (w == 0) { ap_m1 = (A)0; ul_m1 = (A)0; ul_m2 = (A)0; }
            else { ap_m1 = s_xa[ps][w - 1]; ul_m1 = s_xu1[ps][w - 1]; ul_m2 = s_xu2[ps][w - 1]; }
        }
        if (lane == 31) ur_p = (w == nw - 1) ? (A)(rowfull[j] - rf_top) : s_xr[ps][w + 1];
        A Av[CPT], an[CPT], uln[CPT], urn[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) Av[k] = excl + loc[k];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            an[k] = al[k] + Av[k];
            uln[k] = Av[k] + (k == 0 ? ul_m1 : ul[k - 1]);
            urn[k] = Av[k] + (k == CPT - 1 ? ur_p : ur[k + 1]);
        }
        const double rf0d = rowfull[j], rf1d = rowfull[j + 1];
        const A rf1 = (A)rf1d;
        const A yc = (A)(((double)j + 0.5) * inv_nd);
        const A ravg = (A)(0.5 * (rf0d + rf1d));
        const int wi0 = j + x0 - (jt - 1);
        A dlw[CPT + 1];  // DLtot(j + x - 1 + q), sliding window over this thread's columns
#pragma unroll
        for (int q = 0; q <= CPT; ++q) dlw[q] = win_dl[wi0 - 1 + q];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int x = x0 + k;
            if (x >= n) continue;
            const A apm1 = k == 0 ? ap_m1 : al[k - 1];
            const A anm1 = k == 0 ? (ap_m1 + excl) : an[k - 1];
            const A ulnm1 = k == 0 ? (excl + ul_m2) : uln[k - 1];
            const A ulpm1 = k == 0 ? ul_m1 : ul[k - 1];
            const A ulpm2 = k == 0 ? ul_m2 : (k == 1 ? ul_m1 : ul[k - 2]);
            const A urp1 = k == CPT - 1 ? ur_p : ur[k + 1];
            const A Dw = dlw[k + 1], Dwm1 = dlw[k];
            const A Tu = win_tu[wi0 + k - 1];
            const A Tv = win_tv[x - j + jb];
            A R_UV = ulpm1 + (Dw - urp1);
            A R_UVm1 = ulnm1 + (Dw - urn[k]);
            A R_Um1Vm1 = ulpm2 + (Dwm1 - ur[k]);
            if (x == 0) { R_UVm1 = (A)0; R_Um1Vm1 = (A)0; }
            const A bt = R_UVm1;
            const A at = Tu - R_Um1Vm1 + rho[k];
            const A gt = Tv - R_UV;
            if (OUT == OUT_CH8) {
                const A dt = Cr - at - bt - gt;
                double* ch = S.ch8 + (size_t)b * 8 * D.nn + (size_t)j * n + x;
                const size_t nn = D.nn;
                ch[0] = an[k];
                ch[nn] = cc[k] - an[k];
                ch[2 * nn] = Cr - cc[k] - rf1 + an[k];
                ch[3 * nn] = rf1 - an[k];
                ch[4 * nn] = at;
                ch[5 * nn] = bt;
                ch[6 * nn] = gt;
                ch[7 * nn] = dt;
            } else {
                // anchor combination (displacement.py:128-130) with b = cavg-a, d = ravg-a,
                // g = C-cavg-ravg+a, delta_t = C-at-bt-gt; since q1+q3 = (1+x-y, 1-x+y) and
                // q2+q4 = (x+y, x+y) in every case, a's coefficient is (1-2y, 1-2x).
                const A a = (A)0.25 * (apm1 + al[k] + anm1 + an[k]);
                const A cavg = cc[k];
                const A K = cavg + ravg - Cr;
                const A xc = xc0 + (A)k * inv_n, s2 = xc + yc;
                const bool below = yc < xc, near = s2 < (A)1;  // displacement.py:62,67
                const A q3x = below ? xc - yc : (A)0, q3y = below ? (A)0 : yc - xc;
                const A q2x = near ? s2 : (A)1, q2y = near ? (A)0 : s2 - (A)1;
                const A q4x = near ? (A)0 : s2 - (A)1, q4y = near ? s2 : (A)1;
                const A ux = (a * ((A)1 - (A)2 * yc) + cavg * q2x + ravg * q4x - K * q3x + xc * (at + gt) + bt) * inv2m;
                const A uy = (a * ((A)1 - (A)2 * xc) + cavg * q2y + ravg * q4y - K * q3y + at + yc * (Cr - at - gt)) * inv2m;
                UT* o = uf + ((size_t)j * n + x) * 2;
                o[0] = (UT)ux;
                o[1] = (UT)uy;
            }
        }
        if (lane == 31) { s_xa[slot][w] = an[CPT - 1]; s_xu1[slot][w] = uln[CPT - 1]; s_xu2[slot][w] = uln[CPT - 2]; }
        if (lane == 0) s_xr[slot][w] = urn[0];
#pragma unroll
        for (int k = 0; k < CPT; ++k) { al[k] = an[k]; ul[k] = uln[k]; ur[k] = urn[k]; }
    }
}

}  // namespace det
