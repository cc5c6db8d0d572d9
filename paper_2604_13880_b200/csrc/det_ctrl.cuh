// Per-cartogram control step (sm_100a): evaluate + stopping rule + next density LUT.
//
// Runs in the LAST k_row CTA of each cartogram (no separate launch).  It does, on
// the device, what engine.py does on the host between two steps:
//   * background count = n^2 - sum of region counts (raster.py:114-118);
//   * collapse check, first zero-count region (engine.py:147-150);
//   * e_r = |o-w|/max(o,w), epsilon = mean, xi = max (engine.py:83-85,151);
//   * trace row (iteration, epsilon, xi, millis) (engine.py:189-195);
//   * best-state tracking with strict '<' and the three stop tests (engine.py:196-211);
//   * background density (engine.py:162-168) and the residual density LUT
//     rho_r = m*(s_r/o_r)/C - 1, rho_bg = m*bdv/C - 1 consumed by k_sat1/k_sat3
//     (build_density, raster.py:166-184, fused with the residual form).
#pragma once
#include <limits.h>
#include "det_common.cuh"

namespace det {

__global__ void k_init_state(Bufs D) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= D.B) return;
    Carto c;
    memset(&c, 0, sizeof(c));
    c.active = 1;
    c.best_xi = INFINITY;
    c.collapsed = -1;
    c.t_prev = globaltimer();
    D.st[b] = c;
    D.maxspan[b] = 0;
}

// Benchmark helper: continue every cartogram from its current state.
__global__ void k_reactivate(Bufs D) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= D.B) return;
    Carto* c = D.st + b;
    if (c->stop == S_COLLAPSED || c->stop == S_BDV || c->stop == S_NEGINDEX) return;
    if (c->stop != S_RUNNING) c->next_iter = c->res_iter + 1;  // its LUT was built by the control step
    c->active = 1;
    c->stop = S_RUNNING;
    c->final_pending = 0;
}

// cmode -1: background count only; 0: loop evaluation of state next_iter; 1: final re-evaluation
// of the best state.  Executed by one whole CTA (blockDim multiple of 32).
// gate: checked after the first round of count loads is issued (one memory round trip for both).
__device__ void ctrl_body(const Topo& T, const Bufs& D, int b, int cmode, int gate = G_ALWAYS) {
    __shared__ double s_es[32], s_em[32];
    __shared__ long long s_os[32];
    __shared__ int s_fz[32];
    __shared__ int s_cont, s_nbg;
    __shared__ double s_bdv;
    const int t = threadIdx.x, R = T.R, lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
    Carto* st = D.st + b;
    int* acc = D.cnt_acc + (size_t)b * (R + 1);
    int* sc = D.cnt_state + (size_t)b * (R + 1);
    const double* wt = D.weights + (size_t)b * R;
    const double* s = D.stats + (size_t)b * R;
    double* er = D.rerr + (size_t)b * R;
    const bool eval = cmode >= 0;
    // the state and constants the serial section reads, loaded up front with the counts
    const Carto c0 = *st;
    const Params P = D.prm[b];
    int fz = INT_MAX;
    long long osum = 0;
    double es = 0.0, em = -INFINITY;
    for (int r0 = 0; r0 < R; r0 += 4 * blockDim.x) {
        int o[4];
        double wr[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // issue all loads first (latency hiding)
            const int r = r0 + q * blockDim.x + t;
            o[q] = r < R ? __ldcg(acc + r) : 0;
            wr[q] = (eval && r < R) ? wt[r] : 1.0;
        }
        if (r0 == 0 && !(gate == G_ACTIVE ? c0.active != 0 : (gate == G_FINAL ? c0.final_pending != 0 : true))) return;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = r0 + q * blockDim.x + t;
            if (r >= R) continue;
            osum += o[q];
            if (!eval) continue;
            sc[r] = o[q];
            if (o[q] == 0) fz = min(fz, r);
            const double od = (double)o[q];
            const double e = fabs(od - wr[q]) / fmax(od, wr[q]);  // engine.py:84
            er[r] = e;
            es += e;
            em = fmax(em, e);
        }
    }
    // one combined block reduction of (count sum, first zero, error sum, error max)
    osum = warp_sum(osum);
    es = warp_sum(es);
    em = warp_max(em);
    fz = warp_min(fz);
    if (lane == 0) { s_os[w] = osum; s_es[w] = es; s_em[w] = em; s_fz[w] = fz; }
    __syncthreads();
    if (w == 0) {
        long long o2 = lane < nw ? s_os[lane] : 0;
        double e2 = lane < nw ? s_es[lane] : 0.0, m2 = lane < nw ? s_em[lane] : -INFINITY;
        int f2 = lane < nw ? s_fz[lane] : INT_MAX;
        o2 = warp_sum(o2); e2 = warp_sum(e2); m2 = warp_max(m2); f2 = warp_min(f2);
        if (lane == 0) { s_os[0] = o2; s_es[0] = e2; s_em[0] = m2; s_fz[0] = f2; }
    }
    __syncthreads();
    const int nbg = (int)((long long)D.nn - s_os[0]);
    if (t == 0) {
        acc[R] = nbg;
        if (eval) sc[R] = nbg;
    }
    if (!eval) return;
    fz = s_fz[0];
    es = s_es[0];
    em = s_em[0];
    const int it = cmode == 0 ? c0.next_iter : c0.best_iter;
    if (t == 0) {
        s_cont = 0;
        int stop = S_RUNNING;
        if (c0.err & E_NEGIDX) {
            stop = S_NEGINDEX;
            st->res_iter = it;
        } else if (fz < R) {
            stop = S_COLLAPSED;
            st->collapsed = fz;
            st->res_iter = it;
        } else {
            const double eps = es / (double)R, xi = em;
            st->eps = eps;
            st->xi = xi;
            st->res_iter = it;
            if (cmode == 1) {
                st->final_pending = 0;
                st->clamps = 0;  // evaluate() returns a fresh state (engine.py:204-208)
            } else {
                const unsigned long long now = globaltimer();
                const double ms = (double)(now - c0.t_prev) * 1e-6;
                st->t_prev = now;
                if (it < D.trace_cap) {
                    double* tr = D.trace + ((size_t)b * D.trace_cap + it) * 4;
                    tr[0] = (double)it; tr[1] = eps; tr[2] = xi; tr[3] = ms;
                    st->trace_len = it + 1;
                }
                if (xi < c0.best_xi) {
                    st->best_xi = xi;
                    st->best_iter = it;
                    st->best_pending = 1;
                } else {
                    st->best_pending = 0;
                }
                if (xi < P.thr) {
                    stop = S_CONVERGED;
                } else if (it - (xi < c0.best_xi ? it : c0.best_iter) >= P.window) {
                    stop = S_STAGNATION;
                    st->final_pending = 1;
                } else if (it >= P.max_iter) {
                    stop = S_MAXITER;
                }
                // background density of the next step (engine.py:162-168); also built for a
                // stopped state so a benchmark can continue from it (det_bench_iterations)
                const double m = (double)D.nn;
                double bdv;
                if (nbg == 0) bdv = P.mean_density0 * P.mult;
                else if (P.mode == 0) bdv = P.background_mass / (double)nbg;
                else bdv = P.mult * P.S / (m - (double)nbg);
                if (!(bdv > 0.0)) {
                    if (stop == S_RUNNING) stop = S_BDV;  // build_density raises ValueError (raster.py:168-169)
                } else {
                    s_cont = 1;
                    s_bdv = bdv;
                    s_nbg = nbg;
                    st->bdv = bdv;
                    if (stop == S_RUNNING) st->next_iter = it + 1;
                }
            }
        }
        if (stop != S_RUNNING) {
            st->stop = stop;
            st->active = 0;
            if (stop != S_STAGNATION) st->final_pending = 0;
        }
    }
    __syncthreads();
    if (!s_cont) return;
    // total mass C = sum_r (s_r/o_r) o_r + bdv n_bg = S + bdv n_bg (the reference's alpha[-1,-1],
    // integral.py:58, agrees to rounding); residual LUT rho = m d / C - 1
    const double bdv = s_bdv;
    const double m = (double)D.nn;
    const double mc = m / (P.S + bdv * (double)s_nbg);
    double* lut = D.lut + (size_t)b * (R + 1);
    float* lutf = D.lutf + (size_t)b * (R + 1);
    for (int r0 = 0; r0 < R; r0 += 4 * blockDim.x) {
        double sv[4], ov[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = r0 + q * blockDim.x + t;
            sv[q] = r < R ? s[r] : 0.0;
            ov[q] = r < R ? (double)sc[r] : 1.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = r0 + q * blockDim.x + t;
            if (r < R) {  // the label texture holds ranks: LUT indexed by rank
                const double v = mc * (sv[q] / ov[q]) - 1.0;
                const int k = T.region_rank[r];
                lut[k] = v;
                lutf[k] = (float)v;
            }
        }
    }
    if (t == 0) {
        lut[R] = mc * bdv - 1.0;
        lutf[R] = (float)lut[R];
        st->C = P.S + bdv * (double)s_nbg;
    }
}

// The control step as its own kernel, one 1024-thread CTA per cartogram: the evaluation of
// the start state, and each loop iteration's step after k_row (launch_row_ctrl).
__global__ void __launch_bounds__(CTRL_THREADS) k_ctrl(Topo T, Bufs D, int cmode, int gate) {
    ctrl_body(T, D, blockIdx.x + D.b0, cmode, gate);
}

}  // namespace det
