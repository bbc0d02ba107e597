/* Oracle helper (TEST INFRASTRUCTURE ONLY): exact 1-NN parent assignment of
 * the DCI batch build, restating /root/reference/pkg/src/icecache/dci.py:527-543
 *
 *     d2 = cand_sq[None, :] - 2.0 * (block @ cand_rows.T);  nearest = argmin(d2)
 *
 * in fp64 with the operation order the device kernel `nn_parent_kernel`
 * uses: every dot product (and every squared norm) is one sequential chain of
 * fused multiply-adds over the lifted coordinates 0..dim-1, starting from +0.
 * Ties go to the first candidate (np.argmin).  Compile with -mfma
 * -ffp-contract=off so the only fusions are the explicit fma() calls.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static double dot_fma(const double *a, const double *b, int dim) {
    double acc = 0.0;
    for (int t = 0; t < dim; ++t) acc = fma(a[t], b[t], acc);
    return acc;
}

/* pts [np, dim], cands [nc, dim] row-major fp64 lifted rows (tail last). */
void oracle_nn_parents(const double *pts, int64_t np_, const double *cands, int64_t nc,
                       int dim, int32_t *out) {
    double *buf = (double *)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
    for (int64_t j = 0; j < nc; ++j) buf[j] = dot_fma(cands + j * dim, cands + j * dim, dim);
    for (int64_t i = 0; i < np_; ++i) {
        const double *p = pts + i * dim;
        double best = 0.0; int32_t arg = -1;
        for (int64_t j = 0; j < nc; ++j) {
            double d2 = buf[j] - 2.0 * dot_fma(p, cands + j * dim, dim);
            if (arg < 0 || d2 < best) { best = d2; arg = (int32_t)j; }
        }
        out[i] = arg;
    }
    free(buf);
}

/* P-DCI projections dirs[m, dim] . vecs[n, dim] -> out[n, m]; same fma chain
 * as the device (`pdci_project`), restating `self.dirs @ vec` (dci.py:107,113). */
void oracle_project(const double *dirs, int m, const double *vecs, int64_t n, int dim,
                    double *out) {
    for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < m; ++j) out[i * m + j] = dot_fma(dirs + (int64_t)j * dim, vecs + i * dim, dim);
}
