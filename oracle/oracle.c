/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded FP64 CPU implementation of what the ECSIM
 * mass-matrix assembly computes (arXiv 2604.19286, PAPER.md).  It exists to
 * check the CUDA path; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant with paper_2604_19286_b200/ (the product path),
 * and the product path never loads it.
 *
 * Every function cites the passage it follows.  Where the paper is silent
 * the reading is the one listed in DESIGN.md "Readings" (R1..R19, numbered as
 * in SURVEY.md §8(c)).
 *
 * Conventions (R1, R2, R11):
 *   - node g sits at x = g*h; cell c = [c*h, (c+1)*h); nodes = cells per axis,
 *     periodic; linearisation is row-major with axis 0 (x) slowest;
 *   - output layout out[(g*S + slot)*C + comp], S = (2n+1)^3 stencil slots,
 *     slot = ((dx+n)*(2n+1) + (dy+n))*(2n+1) + (dz+n) for the UNWRAPPED node
 *     offset d = g' - g in {-n..n}^3, comp = 3*i + j (C = 9) or 0 (C = 1).
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t n[3];    /* cells = nodes per axis (periodic)                     */
    double h[3];     /* spacing Delta x^mu                                     */
    int32_t x_begin; /* owned cell/node range along axis 0 (whole: 0, n[0])   */
    int32_t x_end;
} or_grid;

typedef struct {
    double qom;   /* q_s / m_s                                                 */
    double dt;    /* Delta t                                                   */
    double c;     /* speed of light (normalised units: 1)                      */
    double sigma; /* constant prefactor sigma of eq_mass_matrix_general        */
} or_species;

enum { OR_OK = 0, OR_ERR_INVALID_ARG = 1, OR_ERR_DOMAIN = 2, OR_ERR_NONFINITE = 3 };

/* ------------------------------------------------------------------------ */
/* Shape functions — PAPER.md:155-168 (eq_shape_bspline, CIC/TSC rules).    */
/* ------------------------------------------------------------------------ */

/* One-dimensional B-spline phi^(n)(t), compactly supported on
 * [-(n+1)/2, (n+1)/2].  n = 1: hat 1 - |t|.  n = 2: the
 * standard quadratic B-spline (reading R3; the paper gives only the order and
 * the support). */
double or_phi(int order, double t)
{
    double a = fabs(t);
    if (order == 1)
        return a <= 1.0 ? 1.0 - a : 0.0;
    if (order == 2) {
        if (a <= 0.5)
            return 0.75 - t * t;
        if (a <= 1.5)
            return 0.5 * (1.5 - a) * (1.5 - a);
        return 0.0;
    }
    return NAN;
}

/* Support of one axis — PAPER.md:166-168.  CIC: nodes {j, j+1} (base 0).
 * TSC: xi < 1/2 -> {j-1, j, j+1} (base -1); xi >= 1/2 -> {j, j+1, j+2}
 * (base 0) (reading R4: the tie xi = 1/2 takes the ">=" branch).
 * w[k] = phi(xi - (base + k)), the distance from the particle to node
 * j + base + k in cell units (eq_shape_bspline). */
int or_support_1d(int order, double xi, int32_t *base, double w[3])
{
    int k;
    if (order == 1)
        *base = 0;
    else if (order == 2)
        *base = (xi >= 0.5) ? 0 : -1;
    else
        return OR_ERR_INVALID_ARG;
    for (k = 0; k < 3; ++k)
        w[k] = (k <= order) ? or_phi(order, xi - (double)(*base + k)) : 0.0;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Rotation-response tensor — PAPER.md:91-96 (eq_alpha_matrix).             */
/*   alpha = (I - C(omega) + omega omega^T) / (1 + |omega|^2),              */
/*   C(omega) u = omega x u.                                                */
/* Row-major: alpha[3*i + j] = alpha^{ij}.                                  */
/* ------------------------------------------------------------------------ */
void or_alpha(const double omega[3], double alpha[9])
{
    double C[9];
    double norm2 = omega[0] * omega[0] + omega[1] * omega[1] + omega[2] * omega[2];
    double d = 1.0 + norm2;
    int i, j;
    /* (omega x u)_i = eps_ijk omega_j u_k, written out as a matrix. */
    C[0] = 0.0;       C[1] = -omega[2]; C[2] = omega[1];
    C[3] = omega[2];  C[4] = 0.0;       C[5] = -omega[0];
    C[6] = -omega[1]; C[7] = omega[0];  C[8] = 0.0;
    for (i = 0; i < 3; ++i)
        for (j = 0; j < 3; ++j)
            alpha[3 * i + j] = ((i == j ? 1.0 : 0.0) - C[3 * i + j] + omega[i] * omega[j]) / d;
}

/* ------------------------------------------------------------------------ */
/* Locating a particle — reading R5: u = x/h (IEEE division), c = floor(u), */
/* xi = u - c.  Positions outside the owned slab are an error, never        */
/* clamped.                                                    */
/* ------------------------------------------------------------------------ */
int or_locate(const or_grid *g, const double x[3], int32_t cell[3], double xi[3])
{
    int mu;
    for (mu = 0; mu < 3; ++mu) {
        double u, c;
        if (!isfinite(x[mu]))
            return OR_ERR_NONFINITE;
        u = x[mu] / g->h[mu];
        c = floor(u);
        xi[mu] = u - c;
        if (mu == 0) {
            if (!(c >= (double)g->x_begin && c < (double)g->x_end))
                return OR_ERR_DOMAIN;
        } else {
            if (!(c >= 0.0 && c < (double)g->n[mu]))
                return OR_ERR_DOMAIN;
        }
        cell[mu] = (int32_t)c;
    }
    return OR_OK;
}

static int check_grid(const or_grid *g, int order)
{
    int mu;
    if (order != 1 && order != 2)
        return OR_ERR_INVALID_ARG;
    for (mu = 0; mu < 3; ++mu) {
        /* reading R11: n >= 2n+1 so distinct unwrapped offsets never alias */
        if (g->n[mu] < 2 * order + 1 || !(g->h[mu] > 0.0))
            return OR_ERR_INVALID_ARG;
    }
    if (g->x_begin < 0 || g->x_end > g->n[0] || g->x_end <= g->x_begin)
        return OR_ERR_INVALID_ARG;
    return OR_OK;
}

static int32_t wrap(int32_t i, int32_t n)
{
    int32_t r = i % n;
    return r < 0 ? r + n : r;
}

/* ------------------------------------------------------------------------ */
/* Binning key — PAPER.md:228 (particles sorted by cell) and PAPER.md:       */
/* 285-296 (eq_group_partition: particles grouped by identical support).    */
/* Reading R12: the key is the support-window base node          */
/* j + b (b = 0 for CIC, b_mu in {-1,0} for TSC), i.e. particles with the    */
/* same key have identical support N_gamma.  Axis 0 is unwrapped and local   */
/* to the slab (bx = c_x + b_x - x_begin + order - 1), axes 1 and 2 wrap.    */
/* ------------------------------------------------------------------------ */
int or_keys(const or_grid *g, int order, int64_t np, const double *pos, const double *q,
            const double *B, uint32_t *key)
{
    int64_t p;
    int rc = check_grid(g, order);
    if (rc)
        return rc;
    for (p = 0; p < np; ++p) {
        int32_t cell[3], base[3], mu;
        double xi[3], w[3];
        rc = or_locate(g, pos + 3 * p, cell, xi);
        if (rc)
            return rc;
        if (!isfinite(q[p]))
            return OR_ERR_NONFINITE;
        if (B && !(isfinite(B[3 * p]) && isfinite(B[3 * p + 1]) && isfinite(B[3 * p + 2])))
            return OR_ERR_NONFINITE;
        for (mu = 0; mu < 3; ++mu)
            or_support_1d(order, xi[mu], &base[mu], w);
        {
            int64_t bx = cell[0] + base[0] - g->x_begin + (order - 1);
            int64_t by = wrap(cell[1] + base[1], g->n[1]);
            int64_t bz = wrap(cell[2] + base[2], g->n[2]);
            key[p] = (uint32_t)((bx * g->n[1] + by) * g->n[2] + bz);
        }
    }
    return OR_OK;
}

int64_t or_nbins(const or_grid *g, int order)
{
    return (int64_t)(g->x_end - g->x_begin + order - 1) * g->n[1] * g->n[2];
}

typedef struct {
    uint32_t key;
    int64_t idx;
} key_idx;

static int cmp_key_idx(const void *a, const void *b)
{
    const key_idx *x = (const key_idx *)a, *y = (const key_idx *)b;
    if (x->key != y->key)
        return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

/* ------------------------------------------------------------------------ */
/* Stable sort by key with K-padding — PAPER.md:228 (sorted by cell),        */
/* PAPER.md:242 (last batch zero-padded), reading R13 (pad records are all   */
/* zero, perm = -1).  Outputs:                                               */
/*   seg_count[b]  number of particles with key b                            */
/*   seg_begin[b]  exclusive scan of ceil(count/K)*K  (nbins + 1 entries)    */
/*   perm[i]       original index of the particle at sorted slot i, or -1    */
/*   rec[8*i..]    {xi_x, xi_y, xi_z, q, Bx, By, Bz, 0} (B = 0 if B == NULL) */
/* perm/rec must hold np + nbins*(K-1) entries.                              */
/* ------------------------------------------------------------------------ */
int or_sort(const or_grid *g, int order, int k_pad, int64_t np, const double *pos,
            const double *q, const double *B, int32_t *perm, int32_t *seg_begin,
            int32_t *seg_count, int64_t *np_padded, double *rec)
{
    int64_t nb, b, p, i;
    uint32_t *key;
    key_idx *ki;
    int rc = check_grid(g, order);
    if (rc)
        return rc;
    if (k_pad < 1)
        return OR_ERR_INVALID_ARG;
    nb = or_nbins(g, order);
    key = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(np > 0 ? np : 1));
    ki = (key_idx *)malloc(sizeof(key_idx) * (size_t)(np > 0 ? np : 1));
    rc = or_keys(g, order, np, pos, q, B, key);
    if (rc) {
        free(key);
        free(ki);
        return rc;
    }
    for (p = 0; p < np; ++p) {
        ki[p].key = key[p];
        ki[p].idx = p;
    }
    qsort(ki, (size_t)np, sizeof(key_idx), cmp_key_idx);
    for (b = 0; b < nb; ++b)
        seg_count[b] = 0;
    for (p = 0; p < np; ++p)
        seg_count[key[p]] += 1;
    seg_begin[0] = 0;
    for (b = 0; b < nb; ++b)
        seg_begin[b + 1] = seg_begin[b] + (seg_count[b] + k_pad - 1) / k_pad * k_pad;
    *np_padded = seg_begin[nb];
    for (i = 0; i < *np_padded; ++i)
        perm[i] = -1;
    /* walk the sorted list: the j-th particle of bin b goes to seg_begin[b]+j */
    i = 0;
    for (b = 0; b < nb; ++b) {
        int32_t j;
        for (j = 0; j < seg_count[b]; ++j, ++i)
            perm[seg_begin[b] + j] = (int32_t)ki[i].idx;
    }
    if (rec) {
        for (i = 0; i < *np_padded; ++i) {
            double *r = rec + 8 * i;
            int k;
            for (k = 0; k < 8; ++k)
                r[k] = 0.0;
            if (perm[i] >= 0) {
                int32_t cell[3];
                int64_t src = perm[i];
                or_locate(g, pos + 3 * src, cell, r);
                r[3] = q[src];
                if (B) {
                    r[4] = B[3 * src];
                    r[5] = B[3 * src + 1];
                    r[6] = B[3 * src + 2];
                }
            }
        }
    }
    free(key);
    free(ki);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* The mass matrix — PAPER.md:84-106:                                        */
/*   eq_mass_matrix_ecsim  (M_s)^{ij}_{gg'} = beta_s/(c V_g) sum_p q_p       */
/*                          alpha_p^{ij} W_pg W_pg'                          */
/*   eq_mass_matrix_general M^{ij}_{gg'} = sigma sum_p s_p^{ij} W_pg W_pg',  */
/*                          s_p^{ij} = q_p alpha_p^{ij}  (scalar: q_p d^ij)  */
/* with omega_p = beta_s B(x_p)/c, beta_s = q_s dt/(2 m_s). */
/* sigma is the caller's (reading R7: not applied implicitly).               */
/* Plain per-particle loop over support-node pairs in input order; the sum  */
/* is the definition written out.  Whole periodic domain only (x_begin = 0, */
/* x_end = n[0]); slab results are compared against slices of it.           */
/* ncomp = 9: tensor (ECSIM), ncomp = 1: scalar (MPM).        */
/* ------------------------------------------------------------------------ */
int or_assemble(const or_grid *g, int order, int ncomp, const or_species *sp, int64_t np,
                const double *pos, const double *q, const double *B, double *out,
                int accumulate)
{
    const int R = order, L = 2 * order + 1, S = L * L * L, N1 = order + 1;
    int64_t nn, p;
    int rc = check_grid(g, order);
    if (rc)
        return rc;
    if (ncomp != 1 && ncomp != 9)
        return OR_ERR_INVALID_ARG;
    if (ncomp == 9 && !B)
        return OR_ERR_INVALID_ARG;
    if (g->x_begin != 0 || g->x_end != g->n[0])
        return OR_ERR_INVALID_ARG;
    nn = (int64_t)g->n[0] * g->n[1] * g->n[2];
    if (!accumulate)
        memset(out, 0, sizeof(double) * (size_t)(nn * S * ncomp));
    for (p = 0; p < np; ++p) {
        int32_t cell[3], base[3];
        double xi[3], w[3][3], s[9];
        int mu, ax, ay, az, bx, by, bz, ij;
        rc = or_locate(g, pos + 3 * p, cell, xi);
        if (rc)
            return rc;
        for (mu = 0; mu < 3; ++mu)
            or_support_1d(order, xi[mu], &base[mu], w[mu]);
        if (ncomp == 9) {
            double beta = sp->qom * sp->dt / 2.0, omega[3], alpha[9];
            for (mu = 0; mu < 3; ++mu)
                omega[mu] = beta * B[3 * p + mu] / sp->c;
            or_alpha(omega, alpha);
            for (ij = 0; ij < 9; ++ij)
                s[ij] = sp->sigma * q[p] * alpha[ij];
        } else {
            s[0] = sp->sigma * q[p];
        }
        for (ax = 0; ax < N1; ++ax)
            for (ay = 0; ay < N1; ++ay)
                for (az = 0; az < N1; ++az) {
                    double Wa = w[0][ax] * w[1][ay] * w[2][az];
                    int64_t ga = ((int64_t)wrap(cell[0] + base[0] + ax, g->n[0]) * g->n[1] +
                                  wrap(cell[1] + base[1] + ay, g->n[1])) * g->n[2] +
                                 wrap(cell[2] + base[2] + az, g->n[2]);
                    for (bx = 0; bx < N1; ++bx)
                        for (by = 0; by < N1; ++by)
                            for (bz = 0; bz < N1; ++bz) {
                                double Wb = w[0][bx] * w[1][by] * w[2][bz];
                                int slot = ((bx - ax + R) * L + (by - ay + R)) * L + (bz - az + R);
                                double ww = Wa * Wb;
                                double *o = out + (ga * S + slot) * ncomp;
                                for (ij = 0; ij < ncomp; ++ij)
                                    o[ij] += s[ij] * ww;
                            }
                }
    }
    return OR_OK;
}

/*
 * or_apply — y (+)= M E, the product of an assembled mass matrix (node-stencil
 * storage above) with a nodal field, as the implicit field equation uses it:
 * (L + sum_s M_s) E = b  (eq_field_eq).  Plain definition:
 *
 *   y[g][i] = sum_{g'} sum_j M^{ij}_{g g'} E[g'][j]
 *           = sum_{slot} sum_j M[g][slot][3 i + j] E[wrap(g + d(slot))][j]   (C = 9)
 *   y[g]    = sum_{slot} M[g][slot] E[wrap(g + d(slot))]                      (C = 1)
 *
 * Whole periodic domain only.  E, y: [nodes][3] (C = 9) or [nodes] (C = 1).
 */
int or_apply(const or_grid *g, int order, int ncomp, const double *M, const double *E, double *y,
             int accumulate)
{
    const int R = order, L = 2 * order + 1, S = L * L * L;
    const int nv = ncomp == 9 ? 3 : 1;
    int64_t gi;
    int rc = check_grid(g, order);
    if (rc)
        return rc;
    if (ncomp != 1 && ncomp != 9)
        return OR_ERR_INVALID_ARG;
    if (g->x_begin != 0 || g->x_end != g->n[0])
        return OR_ERR_INVALID_ARG;
    for (gi = 0; gi < (int64_t)g->n[0] * g->n[1] * g->n[2]; ++gi) {
        int32_t gx = (int32_t)(gi / ((int64_t)g->n[1] * g->n[2]));
        int32_t gy = (int32_t)((gi / g->n[2]) % g->n[1]);
        int32_t gz = (int32_t)(gi % g->n[2]);
        double acc[3] = {0.0, 0.0, 0.0};
        int dx, dy, dz, i, j;
        for (dx = -R; dx <= R; ++dx)
            for (dy = -R; dy <= R; ++dy)
                for (dz = -R; dz <= R; ++dz) {
                    int slot = ((dx + R) * L + (dy + R)) * L + (dz + R);
                    int64_t gn = ((int64_t)wrap(gx + dx, g->n[0]) * g->n[1] + wrap(gy + dy, g->n[1])) * g->n[2] +
                                 wrap(gz + dz, g->n[2]);
                    const double *m = M + (gi * S + slot) * ncomp;
                    for (i = 0; i < nv; ++i)
                        for (j = 0; j < nv; ++j)
                            acc[i] += m[nv * i + j] * E[gn * nv + j];
                }
        for (i = 0; i < nv; ++i)
            y[gi * nv + i] = accumulate ? y[gi * nv + i] + acc[i] : acc[i];
    }
    return OR_OK;
}

/*
 * or_assemble_omp — the same definition (eq_mass_matrix_general) computed by
 * the same per-particle loop as or_assemble, on all host cores, for TIMING the CPU baseline
 * (SURVEY.md §8(c) "An optional OpenMP variant for timing only", §8(d)).  The cells are split
 * into `nslab` x-slabs of at least 3 cells; the particles of a slab (kept in input order) touch
 * only node planes within one cell of the slab, so slabs of the same colour (even / odd index;
 * an odd last slab gets a third colour) never write the same row and run in parallel, one
 * colour after the other.  Deterministic for a given thread count; equal to or_assemble up to
 * the order of the additions (bit-identical on dyadic-lattice inputs).  Whole periodic domain.
 */
int or_assemble_omp(const or_grid *g, int order, int ncomp, const or_species *sp, int64_t np,
                    const double *pos, const double *q, const double *B, double *out, int accumulate,
                    int *threads_used)
{
    const int n0 = g->n[0];
    int nslab = n0 / 3 >= 4 ? (n0 / 3) & ~1 : n0 / 3, c, rc;  /* even when possible: 2 colours */
    int64_t p, *cnt, *idx, *fill;
    const int S = (2 * order + 1) * (2 * order + 1) * (2 * order + 1);
    int64_t nn;
    rc = check_grid(g, order);
    if (rc)
        return rc;
    if (g->x_begin != 0 || g->x_end != n0 || (ncomp != 1 && ncomp != 9) || (ncomp == 9 && !B))
        return OR_ERR_INVALID_ARG;
    if (threads_used)
        *threads_used = 1;
    if (nslab < 2)
        return or_assemble(g, order, ncomp, sp, np, pos, q, B, out, accumulate);
    nn = (int64_t)n0 * g->n[1] * g->n[2];
    if (!accumulate)
        memset(out, 0, sizeof(double) * (size_t)(nn * S * ncomp));
    /* stable bucketing of the particle indices by slab (slab k holds cells [k n0/nslab, ...)) */
    cnt = (int64_t *)calloc((size_t)nslab + 1, sizeof(int64_t));
    fill = (int64_t *)calloc((size_t)nslab + 1, sizeof(int64_t));
    idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(np > 0 ? np : 1));
    for (p = 0; p < np; ++p) {
        int32_t cell[3];
        double xi[3];
        rc = or_locate(g, pos + 3 * p, cell, xi);
        if (rc) {
            free(cnt);
            free(fill);
            free(idx);
            return rc;
        }
        cnt[(int64_t)cell[0] * nslab / n0 + 1] += 1;
    }
    for (c = 0; c < nslab; ++c)
        cnt[c + 1] += cnt[c];
    for (p = 0; p < np; ++p) {
        int32_t cell[3];
        double xi[3];
        int k;
        or_locate(g, pos + 3 * p, cell, xi);
        k = (int)((int64_t)cell[0] * nslab / n0);
        idx[cnt[k] + fill[k]++] = p;
    }
    for (c = 0; c < 3; ++c) {
        int k;
#pragma omp parallel for schedule(dynamic, 1)
        for (k = 0; k < nslab; ++k) {
            int colour = (nslab % 2 == 1 && k == nslab - 1) ? 2 : (k % 2);
            int64_t i;
            if (colour != c)
                continue;
            for (i = cnt[k]; i < cnt[k + 1]; ++i) {
                const int64_t pp = idx[i];
                or_assemble(g, order, ncomp, sp, 1, pos + 3 * pp, q + pp, B ? B + 3 * pp : NULL, out, 1);
            }
        }
    }
#ifdef _OPENMP
    if (threads_used) {
#pragma omp parallel
#pragma omp single
        *threads_used = omp_get_num_threads();
    }
#endif
    free(cnt);
    free(fill);
    free(idx);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: the same particle-to-grid machinery for moment  */
/* deposition, and the grid-to-particle field gather that feeds alpha.      */
/* ------------------------------------------------------------------------ */

/*
 * or_moments — particle moments deposited on the nodes, PAPER.md:591 ("any particle-to-grid
 * scatter operation ... standard charge and current deposition (four quantities per particle in
 * 3D) ... the Implicit Moment Method (ten quantities per particle)"):
 *
 *   mom[g][m] = sigma * sum_p Q_p^m W_pg          (eq_shape_bspline weights)
 *   Q_p = q_p (1, vx, vy, vz)                                              nq = 4  (rho, J)
 *   Q_p = q_p (1, vx, vy, vz, vx vx, vx vy, vx vz, vy vy, vy vz, vz vz)    nq = 10 (implicit
 *         moments: rho, J and the second-moment tensor, upper triangle row-major; reading R20)
 *
 * Plain per-particle loop over the support nodes in input order.  Whole periodic domain.
 * out: [nodes][nq].  v: [np][3].
 */
int or_moments(const or_grid *g, int order, int nq, double sigma, int64_t np, const double *pos,
               const double *q, const double *v, double *out, int accumulate)
{
    const int N1 = order + 1;
    int64_t nn, p;
    int rc = check_grid(g, order);
    if (rc)
        return rc;
    if ((nq != 4 && nq != 10) || !v)
        return OR_ERR_INVALID_ARG;
    if (g->x_begin != 0 || g->x_end != g->n[0])
        return OR_ERR_INVALID_ARG;
    nn = (int64_t)g->n[0] * g->n[1] * g->n[2];
    if (!accumulate)
        memset(out, 0, sizeof(double) * (size_t)(nn * nq));
    for (p = 0; p < np; ++p) {
        int32_t cell[3], base[3];
        double xi[3], w[3][3], Q[10];
        const double *vp = v + 3 * p;
        int mu, ax, ay, az, m;
        rc = or_locate(g, pos + 3 * p, cell, xi);
        if (rc)
            return rc;
        if (!isfinite(q[p]) || !isfinite(vp[0]) || !isfinite(vp[1]) || !isfinite(vp[2]))
            return OR_ERR_NONFINITE;
        for (mu = 0; mu < 3; ++mu)
            or_support_1d(order, xi[mu], &base[mu], w[mu]);
        Q[0] = 1.0;
        Q[1] = vp[0];
        Q[2] = vp[1];
        Q[3] = vp[2];
        Q[4] = vp[0] * vp[0];
        Q[5] = vp[0] * vp[1];
        Q[6] = vp[0] * vp[2];
        Q[7] = vp[1] * vp[1];
        Q[8] = vp[1] * vp[2];
        Q[9] = vp[2] * vp[2];
        for (m = 0; m < nq; ++m)
            Q[m] = sigma * q[p] * Q[m];
        for (ax = 0; ax < N1; ++ax)
            for (ay = 0; ay < N1; ++ay)
                for (az = 0; az < N1; ++az) {
                    double Wa = w[0][ax] * w[1][ay] * w[2][az];
                    int64_t ga = ((int64_t)wrap(cell[0] + base[0] + ax, g->n[0]) * g->n[1] +
                                  wrap(cell[1] + base[1] + ay, g->n[1])) * g->n[2] +
                                 wrap(cell[2] + base[2] + az, g->n[2]);
                    for (m = 0; m < nq; ++m)
                        out[ga * nq + m] += Q[m] * Wa;
                }
    }
    return OR_OK;
}

/*
 * or_gather — a nodal field interpolated to the particle positions, PAPER.md:96 ("B(x_p) being
 * the magnetic field interpolated to the particle position"), with the same shape functions:
 *
 *   Fp[p][i] = sum_g W_pg F[g][i],   i < ncomp      (F: [nodes][ncomp], Fp: [np][ncomp])
 *
 * The nodal field lives on the nodes x_g = g h (reading R1) of the whole periodic domain.
 */
int or_gather(const or_grid *g, int order, int ncomp, int64_t np, const double *pos, const double *F,
              double *Fp)
{
    const int N1 = order + 1;
    int64_t p;
    int rc = check_grid(g, order);
    if (rc)
        return rc;
    if (ncomp < 1 || ncomp > 16)
        return OR_ERR_INVALID_ARG;
    if (g->x_begin != 0 || g->x_end != g->n[0])
        return OR_ERR_INVALID_ARG;
    for (p = 0; p < np; ++p) {
        int32_t cell[3], base[3];
        double xi[3], w[3][3];
        int mu, ax, ay, az, i;
        rc = or_locate(g, pos + 3 * p, cell, xi);
        if (rc)
            return rc;
        for (mu = 0; mu < 3; ++mu)
            or_support_1d(order, xi[mu], &base[mu], w[mu]);
        for (i = 0; i < ncomp; ++i)
            Fp[p * ncomp + i] = 0.0;
        for (ax = 0; ax < N1; ++ax)
            for (ay = 0; ay < N1; ++ay)
                for (az = 0; az < N1; ++az) {
                    double Wa = w[0][ax] * w[1][ay] * w[2][az];
                    int64_t ga = ((int64_t)wrap(cell[0] + base[0] + ax, g->n[0]) * g->n[1] +
                                  wrap(cell[1] + base[1] + ay, g->n[1])) * g->n[2] +
                                 wrap(cell[2] + base[2] + az, g->n[2]);
                    for (i = 0; i < ncomp; ++i)
                        Fp[p * ncomp + i] += Wa * F[ga * ncomp + i];
                }
    }
    return OR_OK;
}
