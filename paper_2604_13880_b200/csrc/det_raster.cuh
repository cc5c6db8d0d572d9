// Advection + rasterisation kernels (sm_100a).
//
// k_region : one CTA per (region, cartogram).  Fuses
//            * advect (displacement.py:209-238): bilinear sample of the u field at
//              every vertex row of the region, clamp to [0,1]^2, clamp count;
//            * the region's bounding-box crop (raster.py:70-78);
//            * even-odd crossing toggles of every ring edge (raster.py:23-61) with the
//              reference's exact float64 op order (explicit _rn intrinsics, no FMA);
//            * the crop flattening of _submask incl. the absorber column and the
//              negative-index case (raster.py:79-90);
//            * per-row toggle sort (smem bitonic) and even-odd pairing into spans.
//            Spans (start, end, rank) go to per-row buckets in HBM.
// k_row    : one CTA per (texture row, cartogram).  Paints spans with smem atomicMin
//            on the region rank (ascending-id first-writer-wins, raster.py:142-146),
//            writes the label row (BACKGROUND=-1) and accumulates per-region pixel
//            counts + background count from run ends (raster.py:110-118).
#pragma once
#include "det_common.cuh"

namespace det {

__device__ __forceinline__ void bitonic_sort_u32(uint32_t* a, int P) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t x = a[i], y = a[ixj];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        a[i] = y;
                        a[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ int lower_bound_u32(const uint32_t* a, int n, uint32_t key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <typename UT>
__device__ __forceinline__ double2 sample_field(const UT* __restrict__ uf, int n, double px, double py) {
    // displacement.py:211-226
    const double nd = (double)n;
    const double gx = px * nd - 0.5, gy = py * nd - 0.5;
    const int ix = clampi((long long)floor(gx), 0, n - 2);
    const int iy = clampi((long long)floor(gy), 0, n - 2);
    const double fx = fmin(fmax(gx - (double)ix, 0.0), 1.0);
    const double fy = fmin(fmax(gy - (double)iy, 0.0), 1.0);
    const size_t o0 = ((size_t)iy * n + ix) * 2, o1 = o0 + (size_t)n * 2;
    const double u00x = (double)uf[o0], u00y = (double)uf[o0 + 1];
    const double u10x = (double)uf[o0 + 2], u10y = (double)uf[o0 + 3];
    const double u01x = (double)uf[o1], u01y = (double)uf[o1 + 1];
    const double u11x = (double)uf[o1 + 2], u11y = (double)uf[o1 + 3];
    const double gxm = 1.0 - fx, gym = 1.0 - fy;
    double2 s;
    s.x = u00x * gxm * gym + u10x * fx * gym + u01x * gxm * fy + u11x * fx * fy;
    s.y = u00y * gxm * gym + u10y * fx * gym + u01y * gxm * fy + u11y * fx * fy;
    return s;
}

template <typename UT>
__global__ void __launch_bounds__(REG_THREADS) k_region(Topo T, Bufs D, int mode, int gate, int src) {
    __shared__ uint32_t s_keys[TOG_CAP];
    __shared__ double s_red[33];
    __shared__ unsigned long long s_redu[33];
    __shared__ int s_tot;

    const int r = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    Carto* st = D.st + b;
    if (!gate_open(st, gate)) return;
    const int n = D.n;
    const double nd = (double)n;
    const int row0 = T.region_row0[r], row1 = T.region_row0[r + 1];
    const size_t ub = (size_t)b * T.n_uniq;

    const double2* pin;
    double2* pout = nullptr;
    bool bestcopy = false;
    if (mode & M_ADVECT) {
        const int cur = st->next_iter - 1;
        pin = ((cur & 1) ? D.pos1 : D.pos0) + ub;
        pout = ((cur & 1) ? D.pos0 : D.pos1) + ub;
        bestcopy = st->best_pending != 0;
    } else {
        pin = (src == 0 ? D.pos0 : (src == 1 ? D.pos1 : D.best)) + ub;
    }
    double2* rowpos = D.rowpos + (size_t)b * T.n_rows;
    const UT* uf = reinterpret_cast<const UT*>(D.uf) + (size_t)b * D.nn * 2;

    // ---- phase A: advect every vertex row of the region, bbox, clamp count ----
    double xmn = INFINITY, xmx = -INFINITY, ymn = INFINITY, ymx = -INFINITY;
    unsigned long long ncl = 0;
    for (int v = row0 + tid; v < row1; v += blockDim.x) {
        const int u = T.row_uniq[v];
        const double2 p = pin[u];
        double2 q = p;
        if (mode & M_ADVECT) {
            const double2 s = sample_field<UT>(uf, n, p.x, p.y);
            const double mx = p.x + s.x, my = p.y + s.y;
            const double cx = fmin(fmax(mx, 0.0), 1.0), cy = fmin(fmax(my, 0.0), 1.0);
            ncl += (cx != mx) + (cy != my);
            q = make_double2(cx, cy);
            if (T.row_owner[v]) {
                pout[u] = q;
                if (bestcopy) D.best[ub + u] = p;
            }
        }
        rowpos[v] = q;
        xmn = fmin(xmn, q.x); xmx = fmax(xmx, q.x);
        ymn = fmin(ymn, q.y); ymx = fmax(ymx, q.y);
    }
    if (mode & M_ADVECT) {
        const unsigned long long tot = block_reduce<0, unsigned long long>(ncl, 0ull, s_redu);
        if (tid == 0 && tot) atomicAdd(&st->clamps, tot);
    }
    if (!(mode & M_RASTER)) return;
    xmn = block_reduce<1, double>(xmn, INFINITY, s_red);
    xmx = block_reduce<2, double>(xmx, -INFINITY, s_red);
    ymn = block_reduce<1, double>(ymn, INFINITY, s_red);
    ymx = block_reduce<2, double>(ymx, -INFINITY, s_red);  // trailing __syncthreads also publishes rowpos

    // ---- region crop (raster.py:70-78) ----
    const int j_off = clampi((long long)ceil(__dsub_rn(__dmul_rn(ymn, nd), 0.5)), 0, n);
    const int j_end = clampi((long long)ceil(__dsub_rn(__dmul_rn(ymx, nd), 0.5)), 0, n);
    const int i_off = clampi((long long)ceil(__dsub_rn(__dmul_rn(xmn, nd), 0.5)), 0, n);
    const int i_end = clampi((long long)ceil(__dsub_rn(__dmul_rn(xmx, nd), 0.5)), 0, n);
    const int rows = max(j_end - j_off, 0), cols = max(i_end - i_off, 0);
    if (rows == 0 || cols == 0) return;
    const long long width = (long long)cols + 1;
    const unsigned long long rank = (unsigned long long)T.region_rank[r];
    const int back = (int)((long long)i_off / width) + 1;  // max rows a negative column can move a toggle up

    int w0 = j_off, wh = rows;
    while (w0 < j_end) {
        const int w1 = min(w0 + wh, j_end);
        if (tid == 0) s_tot = 0;
        __syncthreads();
        // ---- crossings of every ring edge (raster.py:30-61, flattening :86-89) ----
        for (int e = row0 + tid; e < row1; e += blockDim.x) {
            const double2 a = rowpos[e], c = rowpos[T.row_next[e]];
            const double x0 = __dmul_rn(a.x, nd), y0 = __dmul_rn(a.y, nd);
            const double x1 = __dmul_rn(c.x, nd), y1 = __dmul_rn(c.y, nd);
            if (y0 == y1) continue;
            const double ylo = fmin(y0, y1), yhi = fmax(y0, y1);
            const int jlo = clampi((long long)ceil(__dsub_rn(ylo, 0.5)), 0, n);
            const int jhi = clampi((long long)ceil(__dsub_rn(yhi, 0.5)), 0, n);
            if (jhi <= jlo) continue;
            const double slope = __ddiv_rn(__dsub_rn(x1, x0), __dsub_rn(y1, y0));
            const int js = max(jlo, w0);
            const int je = min(jhi, w1 + back);
            for (int j = js; j < je; ++j) {
                const double yc = (double)j + 0.5;
                const double xc = __dadd_rn(x0, __dmul_rn(__dsub_rn(yc, y0), slope));
                const int i0 = clampi((long long)ceil(__dsub_rn(xc, 0.5)), 0, n);
                const long long f = (long long)(j - j_off) * width + (long long)min(i0 - i_off, cols);
                if (f < 0) {  // np.bincount raises on negative entries
                    atomicOr(&st->err, (int)E_NEGIDX);
                    continue;
                }
                const long long dr = f / width;
                const int cc = (int)(f - dr * width);
                if (cc == cols) continue;  // absorber column
                const int dest = j_off + (int)dr;
                if (dest < w0 || dest >= w1) continue;
                const int slot = atomicAdd(&s_tot, 1);
                if (slot < TOG_CAP) s_keys[slot] = ((uint32_t)(dest - w0) << 14) | (uint32_t)(i_off + cc);
            }
        }
        __syncthreads();
        const int tot = s_tot;
        if (tot > TOG_CAP) {
            if (w1 - w0 == 1) {
                if (tid == 0) atomicOr(&st->err, (int)E_TOGGLE_OVF);
                return;
            }
            wh = max(1, (w1 - w0) >> 1);
            __syncthreads();
            continue;
        }
        int P = 1;
        while (P < tot) P <<= 1;
        for (int i = tot + tid; i < P; i += blockDim.x) s_keys[i] = SENT;
        __syncthreads();
        bitonic_sort_u32(s_keys, P);
        // ---- even-odd pairing within each row -> spans [start, end) clipped to the crop ----
        for (int p = tid; p < tot; p += blockDim.x) {
            const uint32_t key = s_keys[p];
            const uint32_t lr = key >> 14;
            const int s0 = lower_bound_u32(s_keys, tot, lr << 14);
            if ((p - s0) & 1) continue;
            const int col = (int)(key & 0x3FFFu);
            const int end = (p + 1 < tot && (s_keys[p + 1] >> 14) == lr) ? (int)(s_keys[p + 1] & 0x3FFFu) : i_end;
            if (end <= col) continue;
            const int row = w0 + (int)lr;
            const size_t rb = (size_t)b * n + row;
            const int slot = atomicAdd(&D.rowcnt[rb], 1);
            if (slot < D.cap)
                D.spans[rb * D.cap + slot] = (rank << 32) | ((unsigned long long)end << 16) | (unsigned long long)col;
            else
                atomicOr(&st->err, (int)E_SPAN_OVF);
        }
        __syncthreads();
        w0 = w1;
        if (tot < TOG_CAP / 4 && wh < rows) wh <<= 1;
    }
}

__global__ void __launch_bounds__(ROW_THREADS) k_row(Topo T, Bufs D, int gate) {
    extern __shared__ uint32_t s_lab[];
    __shared__ int s_c;
    const int j = blockIdx.x, b = blockIdx.y, tid = threadIdx.x, n = D.n;
    Carto* st = D.st + b;
    if (!gate_open(st, gate)) return;
    for (int i = tid; i < n; i += blockDim.x) s_lab[i] = SENT;
    const size_t rb = (size_t)b * n + j;
    if (tid == 0) {
        const int c = D.rowcnt[rb];
        s_c = c;
        D.rowcnt[rb] = 0;
        if (c > D.cap) atomicOr(&st->err, (int)E_SPAN_OVF);
        if (c > 0) atomicMax(&D.maxspan[b], c);
    }
    __syncthreads();
    const int c = min(s_c, D.cap);
    const unsigned long long* sp = D.spans + rb * D.cap;
    for (int s = tid; s < c; s += blockDim.x) {
        const unsigned long long v = sp[s];
        const int lo = (int)(v & 0xFFFFull), hi = (int)((v >> 16) & 0xFFFFull);
        const uint32_t rk = (uint32_t)(v >> 32);
        for (int i = lo; i < hi; ++i) atomicMin(&s_lab[i], rk);
    }
    __syncthreads();
    int* lab = D.labels + (size_t)b * D.nn + (size_t)j * n;
    int* cnt = D.cnt_acc + (size_t)b * (T.R + 1);
    for (int i = tid; i < n; i += blockDim.x) {
        const uint32_t rk = s_lab[i];
        const int L = (rk == SENT) ? -1 : T.rank_region[rk];
        lab[i] = L;
        const int slot = L < 0 ? T.R : L;
        if (i == n - 1 || s_lab[i + 1] != rk) atomicAdd(&cnt[slot], i + 1);
        if (i == 0 || s_lab[i - 1] != rk) atomicAdd(&cnt[slot], -i);
    }
}

// Stage-level advect (displacement.py:229-238) on a float64 field.
__global__ void k_advect_points(const double* __restrict__ uf, int n, const double2* __restrict__ in, int np,
                                double2* __restrict__ out, unsigned long long* clamps) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c = 0;
    if (i < np) {
        const double2 p = in[i];
        const double2 s = sample_field<double>(uf, n, p.x, p.y);
        const double mx = p.x + s.x, my = p.y + s.y;
        const double cx = fmin(fmax(mx, 0.0), 1.0), cy = fmin(fmax(my, 0.0), 1.0);
        c = (cx != mx) + (cy != my);
        out[i] = make_double2(cx, cy);
    }
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(clamps, c);
}

// Stage-level build_density (raster.py:166-184): histogram then gather.
__global__ void k_hist(const int* __restrict__ lab, size_t nn, int R, int* cnt) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x) {
        const int L = lab[i];
        atomicAdd(&cnt[L < 0 ? R : L], 1);
    }
}
__global__ void k_density(const int* __restrict__ lab, size_t nn, int R, const double* __restrict__ stats,
                          const int* __restrict__ cnt, double bdv, double* d) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nn; i += (size_t)gridDim.x * blockDim.x) {
        const int L = lab[i];
        d[i] = L < 0 ? bdv : stats[L] / (double)cnt[L];
    }
}

// Vertex rows of the selected positions (src 0/1/2 = pos0/pos1/best) -> rowpos.
__global__ void k_gather_rows(Topo T, Bufs D, int b, int src) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= T.n_rows) return;
    const size_t ub = (size_t)b * T.n_uniq;
    const double2* p = (src == 0 ? D.pos0 : (src == 1 ? D.pos1 : D.best)) + ub;
    D.rowpos[(size_t)b * T.n_rows + v] = p[T.row_uniq[v]];
}

// Region.area(): signed shoelace over the region's rings (geomodel.py:24-31, 63-65).
__global__ void k_areas(Topo T, Bufs D, const int* __restrict__ ring_start, const int* __restrict__ region_ring0,
                        int b, double* out) {
    __shared__ double s_red[33];
    const int r = blockIdx.x;
    const double2* rp = D.rowpos + (size_t)b * T.n_rows;
    double acc = 0.0;
    for (int q = region_ring0[r]; q < region_ring0[r + 1]; ++q) {
        const int a = ring_start[q], e = ring_start[q + 1];
        if (e - a < 3) continue;
        for (int v = a + threadIdx.x; v < e; v += blockDim.x) {
            const double2 p = rp[v], nx = rp[v + 1 < e ? v + 1 : a];
            acc += p.x * nx.y - nx.x * p.y;
        }
    }
    const double s = block_reduce<0, double>(acc, 0.0, s_red);
    if (threadIdx.x == 0) out[r] = 0.5 * s;
}

}  // namespace det
