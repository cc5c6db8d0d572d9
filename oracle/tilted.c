/*
 * ORACLE (test infrastructure only) -- CPU restatement of the reference's
 * numba-compiled tilted integral-image recurrences.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker / CPU baseline.
 *
 * Follows /root/reference/pkg/src/cartomorph/integral.py:
 *   det_oracle_closed_top_cone  <- _closed_top_cone   (integral.py:65-99)
 *   det_oracle_diag_up_left     <- _diag_up_left      (integral.py:102-112)
 *   det_oracle_diag_up_right    <- _diag_up_right     (integral.py:115-125)
 *
 * Arithmetic order matches the reference expression by expression so the
 * results are bit-identical to the numba build (compile with
 * -ffp-contract=off; see oracle/Makefile).  Arrays are row-major [j][i],
 * h rows by w columns, float64.
 */
#include <stdlib.h>
#include <string.h>

/* Sum over {(i',j'): j' <= j, |i'-i| <= j-j'} for every pixel, using a rolling
 * three-row band padded by h on both sides (zero fill outside the texture). */
int det_oracle_closed_top_cone(const double *d, int h, int w, double *out)
{
    const long pad = h;
    const long width = (long)w + 2 * pad;
    double *buf = (double *)calloc((size_t)(3 * width), sizeof(double));
    if (!buf) return 1;
    double *older = buf, *prev = buf + width, *row = buf + 2 * width;
    for (long j = 0; j < h; ++j) {
        if (j == 0) {
            for (long i = 0; i < w; ++i) row[pad + i] = d[i];
        } else {
            long lo = pad - j - 1;
            if (lo < 1) lo = 1;
            long hi = pad + w + j + 1;
            if (hi > width - 1) hi = width - 1;
            for (long c = lo; c < hi; ++c) {
                double v = prev[c - 1] + prev[c + 1] - older[c];
                long i = c - pad;
                if (i >= 0 && i < w) v += d[j * w + i] + d[(j - 1) * w + i];
                row[c] = v;
            }
        }
        memcpy(out + j * w, row + pad, (size_t)w * sizeof(double));
        double *t = older;
        older = prev;
        prev = row;
        row = t;
    }
    free(buf);
    return 0;
}

/* out(i,j) = d(i,j) + d(i-1,j-1) + ... (half line toward the upper left). */
int det_oracle_diag_up_left(const double *d, int h, int w, double *out)
{
    for (int i = 0; i < w; ++i) out[i] = d[i];
    for (long j = 1; j < h; ++j) {
        out[j * w] = d[j * w];
        for (long i = 1; i < w; ++i) out[j * w + i] = d[j * w + i] + out[(j - 1) * w + i - 1];
    }
    return 0;
}

/* out(i,j) = d(i,j) + d(i+1,j-1) + ... (half line toward the upper right). */
int det_oracle_diag_up_right(const double *d, int h, int w, double *out)
{
    for (int i = 0; i < w; ++i) out[i] = d[i];
    for (long j = 1; j < h; ++j) {
        out[j * w + w - 1] = d[j * w + w - 1];
        for (long i = 0; i < w - 1; ++i) out[j * w + i] = d[j * w + i] + out[(j - 1) * w + i + 1];
    }
    return 0;
}
