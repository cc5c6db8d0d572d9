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

template <int CPT, int SRC>
__device__ __forceinline__ void load_rho(const Bufs& D, const SatSrc& S, int R, int b, int j, int x0,
                                         double (&rho)[CPT]) {
    const int n = D.n;
    if (x0 >= n) {
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = 0.0;
        return;
    }
    if (SRC == SRC_LABELS) {
        const int* lab = D.labels + (size_t)b * D.nn + (size_t)j * n + x0;
        const double* lut = D.lut + (size_t)b * (R + 1);
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
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = __ldg(lut + (L[k] < 0 ? R : L[k]));
    } else {
        const double* d = S.d + (size_t)b * D.nn + (size_t)j * n + x0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) rho[k] = __dadd_rn(__dmul_rn(d[k], S.scale), S.offset);
    }
}

// In-place inclusive prefix of a[0..len) in shared memory by the whole CTA.
__device__ void block_prefix_smem(double* a, int len, double* sm) {
    const int nt = blockDim.x;
    const int per = (len + nt - 1) / nt;
    const int s = min(len, threadIdx.x * per), e = min(len, s + per);
    double loc = 0.0;
    for (int i = s; i < e; ++i) loc += a[i];
    double tot;
    double run = block_excl_scan(loc, sm, &tot);
    for (int i = s; i < e; ++i) {
        run += a[i];
        a[i] = run;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------------
// Per-band sums, x-prefixed:  CS_b(x) = sum_{j in band, i<=x} rho,
// DG_b(v) = sum_{j in band, i-j<=v} rho (compact index q = v + jb, q in [0, n+H-1)),
// AD_b(w) = sum_{j in band, i+j<=w} rho (compact index q = w - jt).  Outside the
// compact range the prefixes are 0 (below) or the band total (above).
template <int CPT, int SRC>
__global__ void k_sat1(Topo T, Bufs D, SatSrc S, int gate) {
    extern __shared__ double s_part[];  // dg[L] | ad[L]
    __shared__ double s_w[3][32];
    __shared__ double s_bd[3][32];
    __shared__ double s_ba[3][32];
    __shared__ double s_red[33];
    const int band = blockIdx.x, b = blockIdx.y, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, L = n + H - 1;
    const int x0 = t * CPT;
    const size_t bb = (size_t)b * D.nb + band;
    double* dg = s_part;
    double* ad = s_part + L;
    double cs[CPT], pd[CPT], pa[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) cs[k] = pd[k] = pa[k] = 0.0;

    for (int j = jt; j <= jb; ++j) {
        const int slot = (j - jt) % 3, ps = (j - jt + 2) % 3;
        double rho[CPT];
        load_rho<CPT, SRC>(D, S, T.R, b, j, x0, rho);
        double ts = 0.0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) ts += rho[k];
        ts = warp_sum(ts);
        if (lane == 0) s_w[slot][w] = ts;
        __syncthreads();
        double left = __shfl_up_sync(FULL, pd[CPT - 1], 1);
        double right = __shfl_down_sync(FULL, pa[0], 1);
        if (lane == 0) left = (w == 0 || j == jt) ? 0.0 : s_bd[ps][w - 1];
        if (lane == 31) right = (w == nw - 1 || j == jt) ? 0.0 : s_ba[ps][w + 1];
        double nd_[CPT], na_[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            nd_[k] = rho[k] + (k == 0 ? left : pd[k - 1]);
            na_[k] = rho[k] + (k == CPT - 1 ? right : pa[k + 1]);
            cs[k] += rho[k];
        }
        if (t == 0) {
            double s = 0.0;
            for (int q = 0; q < nw; ++q) s += s_w[slot][q];
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
        csum += x < n ? cs[k] : 0.0;
    }
    double tot;
    double run = block_excl_scan(csum, s_red, &tot);
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        run += cs[k];
        if (x < n) D.cs[bb * n + x] = run;
    }
    block_prefix_smem(dg, L, s_red);
    block_prefix_smem(ad, L, s_red);
    for (int q = t; q < L; q += blockDim.x) {
        D.dgc[bb * L + q] = dg[q];
        D.adc[bb * L + q] = ad[q];
    }
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
    const int b = blockIdx.y, t = threadIdx.x, lx = t & 31, g = t >> 5, G = blockDim.x >> 5;
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
template <int CPT, int SRC, typename UT, int OUT>
__global__ void k_sat3(Topo T, Bufs D, SatSrc S, int gate) {
    extern __shared__ double sm[];
    __shared__ double s_w[3][32];
    __shared__ double s_xa[3][32], s_xu1[3][32], s_xu2[3][32], s_xr[3][32];
    const int band = blockIdx.x, b = blockIdx.y, t = threadIdx.x;
    const int lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
    if (!gate_open(D.st + b, gate)) return;
    const int n = D.n, H = D.H, jt = band * H, jb = jt + H - 1, M = 2 * n - 1;
    const int x0 = t * CPT;
    const size_t bb = (size_t)b * D.nb + band;
    const int WN = n + H;
    double* win_dl = sm;            // DLtot(w), w in [jt-1, jb+n-1]  -> [w-(jt-1)]
    double* win_tu = sm + WN;       // Tu(w),    w in [jt-1, jb+n-2]  -> [w-(jt-1)]
    double* win_tv = sm + 2 * WN;   // Tv(v),    v in [-jb, n-1-jt]   -> [v+jb]
    const double* rowfull = D.rowfull + (size_t)b * (n + 1);
    const double* adT = D.adT + (size_t)b * M;
    const double* dgT = D.dgT + (size_t)b * M;
    const double* csT = D.csT + (size_t)b * n;

    // ---- carries (k_sat2) ----
    for (int q = t; q < WN; q += blockDim.x) {
        win_dl[q] = (jt == 0 && q == 0) ? 0.0 : D.adSc[bb * WN + q];  // DLtot(-1) = 0
        const int wq = jt - 1 + q;
        win_tu[q] = (wq >= 0 && wq < M) ? adT[wq] : 0.0;
        const int iv = q - jb + n - 1;  // Tv index of v = q - jb
        win_tv[q] = (iv >= 0 && iv < M) ? dgT[iv] : 0.0;
    }
    double ul[CPT], al[CPT], cfe[CPT], cfi[CPT], ur[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int x = x0 + k;
        const bool in = x < n;
        al[k] = in ? D.csX[bb * n + x] : 0.0;
        ul[k] = in ? D.dgXc[bb * n + x] : 0.0;
        cfi[k] = in ? csT[x] : 0.0;
        cfe[k] = (in && x > 0) ? csT[x - 1] : 0.0;
        ur[k] = 0.0;
    }
    if (lane == 31) {  // boundary values of "row jt-1" = carries
        s_xa[2][w] = al[CPT - 1];
        s_xu1[2][w] = ul[CPT - 1];
        s_xu2[2][w] = ul[CPT - 2];
    }
    if (lane == 0) s_xr[2][w] = 0.0;
    __syncthreads();

    const double rf_top = rowfull[jt];
    const double Cr = rowfull[n];
    const double nd = (double)n;
    const double inv2m = S.outscale != 0.0 ? S.outscale : 0.5 / (nd * nd);
    UT* uf = reinterpret_cast<UT*>(D.uf) + (size_t)b * D.nn * 2;

    for (int j = jt; j <= jb; ++j) {
        const int slot = (j - jt) % 3, ps = (j - jt + 2) % 3;
        double rho[CPT];
        load_rho<CPT, SRC>(D, S, T.R, b, j, x0, rho);
        double loc[CPT];
        double run = 0.0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) { run += rho[k]; loc[k] = run; }
        const double tsum = run;
        const double winc = warp_incl_scan(tsum);
        if (lane == 31) s_w[slot][w] = winc;
        __syncthreads();
        double off = 0.0;
        for (int q = 0; q < w; ++q) off += s_w[slot][q];
        const double excl = off + winc - tsum;  // A(j, x0-1)
        double ap_m1 = __shfl_up_sync(FULL, al[CPT - 1], 1);
        double ul_m1 = __shfl_up_sync(FULL, ul[CPT - 1], 1);
        double ul_m2 = __shfl_up_sync(FULL, ul[CPT - 2], 1);
        double ur_p = __shfl_down_sync(FULL, ur[0], 1);
        if (lane == 0) {
            if (w == 0) { ap_m1 = 0.0; ul_m1 = 0.0; ul_m2 = 0.0; }
            else { ap_m1 = s_xa[ps][w - 1]; ul_m1 = s_xu1[ps][w - 1]; ul_m2 = s_xu2[ps][w - 1]; }
        }
        if (lane == 31) ur_p = (w == nw - 1) ? (rowfull[j] - rf_top) : s_xr[ps][w + 1];
        double A[CPT], an[CPT], uln[CPT], urn[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) A[k] = excl + loc[k];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            an[k] = al[k] + A[k];
            uln[k] = A[k] + (k == 0 ? ul_m1 : ul[k - 1]);
            urn[k] = A[k] + (k == CPT - 1 ? ur_p : ur[k + 1]);
        }
        const double rf0 = rowfull[j], rf1 = rowfull[j + 1];
        const double yc = ((double)j + 0.5) / nd;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int x = x0 + k;
            if (x >= n) continue;
            const double apm1 = k == 0 ? ap_m1 : al[k - 1];
            const double anm1 = k == 0 ? (ap_m1 + excl) : an[k - 1];
            const double ulnm1 = k == 0 ? (excl + ul_m2) : uln[k - 1];
            const double ulpm1 = k == 0 ? ul_m1 : ul[k - 1];
            const double ulpm2 = k == 0 ? ul_m2 : (k == 1 ? ul_m1 : ul[k - 2]);
            const double urp1 = k == CPT - 1 ? ur_p : ur[k + 1];
            const int wi = j + x - (jt - 1);
            const double Dw = win_dl[wi], Dwm1 = win_dl[wi - 1];
            const double Tu = win_tu[wi - 1];
            const double Tv = win_tv[x - j + jb];
            double R_UV = ulpm1 + (Dw - urp1);
            double R_UVm1 = ulnm1 + (Dw - urn[k]);
            double R_Um1Vm1 = ulpm2 + (Dwm1 - ur[k]);
            if (x == 0) { R_UVm1 = 0.0; R_Um1Vm1 = 0.0; }
            const double bt = R_UVm1;
            const double at = Tu - R_Um1Vm1 + rho[k];
            const double gt = Tv - R_UV;
            const double dt = Cr - at - bt - gt;
            if (OUT == OUT_CH8) {
                double* ch = S.ch8 + (size_t)b * 8 * D.nn + (size_t)j * n + x;
                const size_t nn = D.nn;
                ch[0] = an[k];
                ch[nn] = cfi[k] - an[k];
                ch[2 * nn] = Cr - cfi[k] - rf1 + an[k];
                ch[3 * nn] = rf1 - an[k];
                ch[4 * nn] = at;
                ch[5 * nn] = bt;
                ch[6 * nn] = gt;
                ch[7 * nn] = dt;
            } else {
                const double a = 0.25 * (apm1 + al[k] + anm1 + an[k]);
                const double cavg = 0.5 * (cfe[k] + cfi[k]), ravg = 0.5 * (rf0 + rf1);
                const double bS = cavg - a, dS = ravg - a, gS = Cr - cavg - ravg + a;
                const double xc = ((double)x + 0.5) / nd;
                double q1x, q1y, q3x, q3y, q2x, q2y, q4x, q4y;  // displacement.py:56-74
                if (yc < xc) { q1x = 1.0; q1y = 1.0 + yc - xc; q3x = xc - yc; q3y = 0.0; }
                else { q1x = 1.0 - yc + xc; q1y = 1.0; q3x = 0.0; q3y = yc - xc; }
                if (xc + yc < 1.0) { q2x = xc + yc; q2y = 0.0; q4x = 0.0; q4y = xc + yc; }
                else { q2x = 1.0; q2y = xc + yc - 1.0; q4x = xc + yc - 1.0; q4y = 1.0; }
                const double ux = (a * q1x + bS * q2x + gS * q3x + dS * q4x + at * xc + bt + gt * xc) * inv2m;
                const double uy = (a * q1y + bS * q2y + gS * q3y + dS * q4y + at + bt * yc + dt * yc) * inv2m;
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
