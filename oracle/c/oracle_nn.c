/* Oracle helper (TEST INFRASTRUCTURE ONLY): exact 1-NN parent assignment of
 * the DCI batch build, restating /root/reference/pkg/src/icecache/dci.py:527-543
 *
 *     d2 = cand_sq[None, :] - 2.0 * (block @ cand_rows.T);  nearest = argmin(d2)
 *
 * in fp64 with the operation order the device kernel `nn_parent_kernel`
 * uses: every dot product (and every squared norm) is one sequential chain of
 * fused multiply-adds over the lifted coordinates 0..dim-1, starting from +0.
 * Ties go to the first candidate (np.argmin).  The loops run over candidates
 * in the innermost position so the compiler vectorizes ACROSS independent
 * dot products; each individual chain keeps its sequential order.
 * Compile with -ffp-contract=off so the only fusions are the fma() calls.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define PB 4

void oracle_nn_parents(const double *pts, int64_t np_, const double *cands, int64_t nc,
                       int dim, int32_t *out) {
    double *csq = (double *)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
    double *ct = (double *)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1) * dim);
    double *acc = (double *)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1) * PB);
    for (int64_t j = 0; j < nc; ++j) {
        double a = 0.0;
        for (int t = 0; t < dim; ++t) {
            double c = cands[j * dim + t];
            a = fma(c, c, a);
            ct[(int64_t)t * nc + j] = c;
        }
        csq[j] = a;
    }
    for (int64_t i0 = 0; i0 < np_; i0 += PB) {
        int nb = (int)((np_ - i0) < PB ? (np_ - i0) : PB);
        for (int b = 0; b < nb; ++b)
            for (int64_t j = 0; j < nc; ++j) acc[b * nc + j] = 0.0;
        for (int t = 0; t < dim; ++t) {
            const double *crow = ct + (int64_t)t * nc;
            for (int b = 0; b < nb; ++b) {
                const double pv = pts[(i0 + b) * dim + t];
                double *ab = acc + b * nc;
                for (int64_t j = 0; j < nc; ++j) ab[j] = fma(pv, crow[j], ab[j]);
            }
        }
        for (int b = 0; b < nb; ++b) {
            double best = 0.0;
            int32_t arg = -1;
            for (int64_t j = 0; j < nc; ++j) {
                double d2 = csq[j] - 2.0 * acc[b * nc + j];
                if (arg < 0 || d2 < best) { best = d2; arg = (int32_t)j; }
            }
            out[i0 + b] = arg;
        }
    }
    free(csq);
    free(ct);
    free(acc);
}

/* P-DCI projections dirs[m, dim] . vecs[n, dim] -> out[n, m]; same fma chain
 * as the device (`pdci_visit`), restating `self.dirs @ vec` (dci.py:107,113). */
void oracle_project(const double *dirs, int m, const double *vecs, int64_t n, int dim,
                    double *out) {
    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < m; ++j) {
            double a = 0.0;
            for (int t = 0; t < dim; ++t) a = fma(dirs[(int64_t)j * dim + t], vecs[i * dim + t], a);
            out[i * m + j] = a;
        }
}

/* Search distance in fp32 with the device's exact operation order
 * (csrc/icb.cuh: lane_sq4 / warp_sum_butterfly / d2_finish): lane l owns
 * dims 4l..4l+3, s_l = fma(d3,d3, fma(d2,d2, fma(d1,d1, d0*d0))), lanes are
 * combined by the xor butterfly 16, 8, 4, 2, 1 with plain adds, and
 * d2 = fma(dt, dt, f) with dt = tail - q_tail.  Restates dci.py:311-312
 * (sum of squared lifted differences).  rows [n][128] fp32 (zero padded). */
void oracle_d2_fp32(const float *rows, const float *tail, int64_t n, const float *q, float q_tail,
                    float *out) {
    for (int64_t r = 0; r < n; ++r) {
        const float *p = rows + r * 128;
        float s[32];
        for (int l = 0; l < 32; ++l) {
            float d0 = p[4 * l] - q[4 * l], d1 = p[4 * l + 1] - q[4 * l + 1];
            float d2 = p[4 * l + 2] - q[4 * l + 2], d3 = p[4 * l + 3] - q[4 * l + 3];
            float a = d0 * d0;
            a = fmaf(d1, d1, a);
            a = fmaf(d2, d2, a);
            a = fmaf(d3, d3, a);
            s[l] = a;
        }
        for (int w = 16; w >= 1; w >>= 1)
            for (int l = 0; l < w; ++l) s[l] = s[l] + s[l + w];
        float dt = tail[r] - q_tail;
        out[r] = fmaf(dt, dt, s[0]);
    }
}
