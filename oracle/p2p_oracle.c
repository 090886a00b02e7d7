/*
 * oracle/p2p_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle of the MLFMA near-field (P2P)
 * operator with the paper's data-redundancy layout (arXiv 2511.21535).
 *
 * *** TEST INFRASTRUCTURE, NOT PRODUCT CODE. ***
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may load
 * this library.  It shares NO code, header, table or constant generator with the CUDA path
 * (paper_2511_21535_b200/csrc); neither side includes or links the other.
 *
 * Citations: P:Lnnn = /root/reference/PAPER.md line nnn; S:Lnnn = SPEC.md line nnn; "C<k>" = the
 * reading with that number in DESIGN.md §3 (taken from SURVEY.md §8c).
 *
 * What it computes ("direct particle-to-particle interactions within neighboring cells";
 * P:L211 "all 9t^2 neighboring patterns"; "27 (E2 neighbors)"; P:L336-338 the indexing and
 * redundant layouts):
 *   gravity   : phi_i = - sum_{j != i} m_j / sqrt(r^2 + eps^2),
 *               a_i   =   sum_j     m_j d_ij / (r^2 + eps^2)^{3/2},   d_ij = x_j + S - x_i   (C1, C3)
 *               over every j in the E2 (3^3 box) neighbourhood of i's leaf box, S the box-level
 *               periodic image shift (C4, C5).
 *   helmholtz : y_i = sum_{q adjacent} w(p_i, q) x_q, w = G(r) Delta^2 off-diagonal, the Richmond disk
 *               self term on the diagonal, G(r) = (i/4) H0^(1)(k r)  (C15).
 * plus every data structure the method builds on the way (keys, stable sort permutation, box table,
 * neighbour CSR, redundant buffer), which the GPU must reproduce bit-exactly.
 *
 * Parity pins (tests/test_oracle_*.py): closed forms, brute force on tiny inputs, Newton's third law,
 * library Bessel functions (scipy), the worked examples of SURVEY §8c.  Everything here is fp64
 * IEEE; build with -ffp-contract=off -fno-fast-math so no FMA contraction changes a rounding
 * (C6, C11).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* --------------------------------------------------------------------------------------------- */
/* a1: binning (C6) and Morton keys (C7)                                                          */
/* --------------------------------------------------------------------------------------------- */

/* ib_d = floor((x_d - lo_d) / h) in fp64 with IEEE divide; out-of-domain is an error, never clamped.
 * Returns -1 on success, else the index of the first offending particle. */
int64_t orc_bin(int dim, int64_t n, const double *pos, double h, const double *lo, const int32_t *nbox,
                int32_t *ib)
{
    for (int64_t i = 0; i < n; ++i) {
        for (int d = 0; d < dim; ++d) {
            double q = (pos[i * dim + d] - lo[d]) / h;
            double f = floor(q);
            if (!(f >= 0.0 && f < (double)nbox[d])) return i;
            ib[i * dim + d] = (int32_t)f;
        }
    }
    return -1;
}

/* bits per dimension: smallest nb with 2^nb >= max_d nbox_d */
int orc_bits_per_dim(int dim, const int32_t *nbox)
{
    int32_t m = 1;
    for (int d = 0; d < dim; ++d) if (nbox[d] > m) m = nbox[d];
    int nb = 0;
    while ((1 << nb) < m) ++nb;
    return nb;
}

/* Morton interleave, the naive bit loop: bit dim*k + d of the key = bit k of coordinate d
 * (3D: bit 3k = x_k, 3k+1 = y_k, 3k+2 = z_k; 2D: bit 2k = x_k, 2k+1 = y_k) -- C7. */
uint32_t orc_morton(int dim, int nb, const int32_t *c)
{
    uint32_t key = 0;
    for (int k = 0; k < nb; ++k)
        for (int d = 0; d < dim; ++d)
            key |= (uint32_t)((c[d] >> k) & 1) << (dim * k + d);
    return key;
}

/* inverse of orc_morton */
void orc_demorton(int dim, int nb, uint32_t key, int32_t *c)
{
    for (int d = 0; d < dim; ++d) c[d] = 0;
    for (int k = 0; k < nb; ++k)
        for (int d = 0; d < dim; ++d)
            c[d] |= (int32_t)((key >> (dim * k + d)) & 1u) << k;
}

/* --------------------------------------------------------------------------------------------- */
/* a2: stable sort by key (C8) -- sorting (key, input index) pairs lexicographically IS the stable  */
/* sort by key.                                                                                    */
/* --------------------------------------------------------------------------------------------- */
static int cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

void orc_stable_sort(int64_t n, const uint32_t *key, uint32_t *skey, uint32_t *perm)
{
    uint64_t *kv = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) kv[i] = ((uint64_t)key[i] << 32) | (uint64_t)i;
    qsort(kv, (size_t)n, sizeof(uint64_t), cmp_u64);
    for (int64_t i = 0; i < n; ++i) {
        skey[i] = (uint32_t)(kv[i] >> 32);
        perm[i] = (uint32_t)(kv[i] & 0xffffffffu);
    }
    free(kv);
}

/* --------------------------------------------------------------------------------------------- */
/* a4: box table from run heads of the sorted keys (C9).  Returns B.                               */
/* --------------------------------------------------------------------------------------------- */
int64_t orc_box_table(int64_t n, const uint32_t *skey, uint32_t *bkey, uint32_t *bstart)
{
    int64_t B = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (i == 0 || skey[i] != skey[i - 1]) {
            bkey[B] = skey[i];
            bstart[B] = (uint32_t)i;
            ++B;
        }
    }
    bstart[B] = (uint32_t)n;
    return B;
}

static int64_t find_box(int64_t B, const uint32_t *bkey, uint32_t key)
{
    int64_t lo = 0, hi = B - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (bkey[mid] == key) return mid;
        if (bkey[mid] < key) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* One stencil step in one dimension (C4, C5): neighbour coordinate c+delta, wrapped when periodic.
 * *shift receives the box-level image of the SOURCE relative to the target: +L when the neighbour
 * wraps past the upper face (index n -> 0), -L past the lower face (-1 -> n-1), else 0.
 * Returns 0 if the neighbour does not exist (open dimension, outside the grid). */
static int step_dim(int32_t c, int delta, int32_t n, int periodic, double L, int32_t *out, double *shift)
{
    int32_t v = c + delta;
    *shift = 0.0;
    if (v < 0) {
        if (!periodic) return 0;
        v += n;
        *shift = -L;
    } else if (v >= n) {
        if (!periodic) return 0;
        v -= n;
        *shift = L;
    }
    *out = v;
    return 1;
}

/* --------------------------------------------------------------------------------------------- */
/* Gravity structures: a1..a5 in one call.                                                         */
/*   key[n], skey[n], perm[n], bkey[<=n], bstart[<=n+1], nbr_off[<=n+1], nbr_box[<=27n],           */
/*   nbr_slot[<=27n], red_off[<=n+1] (u64).  counts = {B, n_nbr, R, I}.                            */
/* Neighbour order (C10): ascending stencil slot s = 9(dz+1) + 3(dy+1) + (dx+1); empty and         */
/* out-of-domain neighbours omitted.                                                               */
/* Returns -1 on success, else the first out-of-domain particle index.                             */
/* --------------------------------------------------------------------------------------------- */
int64_t orc_gravity_structs(int64_t n, const double *pos, double h, const double *lo, const int32_t *nbox,
                            uint32_t periodic, uint32_t *key, uint32_t *skey, uint32_t *perm, uint32_t *bkey,
                            uint32_t *bstart, uint32_t *nbr_off, uint32_t *nbr_box, uint8_t *nbr_slot,
                            uint64_t *red_off, int64_t *counts)
{
    int32_t *ib = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)(n > 0 ? n : 1));
    int64_t bad = orc_bin(3, n, pos, h, lo, nbox, ib);
    if (bad >= 0) { free(ib); return bad; }
    int nb = orc_bits_per_dim(3, nbox);
    for (int64_t i = 0; i < n; ++i) key[i] = orc_morton(3, nb, &ib[3 * i]);
    orc_stable_sort(n, key, skey, perm);
    int64_t B = orc_box_table(n, skey, bkey, bstart);
    int64_t e = 0;
    uint64_t R = 0, I = 0;
    for (int64_t b = 0; b < B; ++b) {
        int32_t c[3];
        orc_demorton(3, nb, bkey[b], c);
        nbr_off[b] = (uint32_t)e;
        red_off[b] = R;
        uint64_t nsrc = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int slot = 9 * (dz + 1) + 3 * (dy + 1) + (dx + 1);
                    int32_t nc[3];
                    double sh[3];
                    int dd[3] = {dx, dy, dz};
                    int ok = 1;
                    for (int d = 0; d < 3; ++d)
                        ok &= step_dim(c[d], dd[d], nbox[d], (periodic >> d) & 1u, (double)nbox[d] * h, &nc[d],
                                       &sh[d]);
                    if (!ok) continue;
                    int64_t k = find_box(B, bkey, orc_morton(3, nb, nc));
                    if (k < 0) continue;
                    nbr_box[e] = (uint32_t)k;
                    nbr_slot[e] = (uint8_t)slot;
                    ++e;
                    nsrc += bstart[k + 1] - bstart[k];
                }
        R += nsrc;
        I += nsrc * (uint64_t)(bstart[b + 1] - bstart[b]);
    }
    nbr_off[B] = (uint32_t)e;
    red_off[B] = R;
    counts[0] = B;
    counts[1] = e;
    counts[2] = (int64_t)R;
    counts[3] = (int64_t)I;
    free(ib);
    return -1;
}

/* image shift of stencil slot `slot` seen from box with coordinates c (C5) */
static void slot_shift(int slot, const int32_t *c, const int32_t *nbox, uint32_t periodic, double h, double *S)
{
    int dd[3] = {slot % 3 - 1, (slot / 3) % 3 - 1, slot / 9 - 1};
    for (int d = 0; d < 3; ++d) {
        int32_t v;
        if (!step_dim(c[d], dd[d], nbox[d], (periodic >> d) & 1u, (double)nbox[d] * h, &v, &S[d])) S[d] = 0.0;
    }
}

/* box origin o_d = fma(ib_d, h, lo_d) (C11: an explicit fma on both sides) */
static void box_origin(const int32_t *c, double h, const double *lo, double *o)
{
    for (int d = 0; d < 3; ++d) o[d] = fma((double)c[d], h, lo[d]);
}

/* --------------------------------------------------------------------------------------------- */
/* a6: the redundant buffer (C11).  For target box b and each neighbour (k, s) in CSR order, the    */
/* records of box k in sorted order, rebased to b's origin:                                        */
/*   red = { fl_p(((double)x_j + S_x) - o_bx), ..y.., ..z.., m_j }                                 */
/* `prec` 0 = fp32 (float[4] records), 1 = fp64 (double[4]).  `pos`/`mass` are the working-precision */
/* inputs promoted to double, in INPUT order.                                                       */
/* --------------------------------------------------------------------------------------------- */
void orc_gravity_red(int prec, int64_t B, const double *pos, const double *mass, double h, const double *lo,
                     const int32_t *nbox, uint32_t periodic, const uint32_t *perm, const uint32_t *bkey,
                     const uint32_t *bstart, const uint32_t *nbr_off, const uint32_t *nbr_box,
                     const uint8_t *nbr_slot, const uint64_t *red_off, void *red)
{
    int nb = orc_bits_per_dim(3, nbox);
    for (int64_t b = 0; b < B; ++b) {
        int32_t c[3];
        double o[3];
        orc_demorton(3, nb, bkey[b], c);
        box_origin(c, h, lo, o);
        uint64_t r = red_off[b];
        for (uint32_t e = nbr_off[b]; e < nbr_off[b + 1]; ++e) {
            double S[3];
            slot_shift(nbr_slot[e], c, nbox, periodic, h, S);
            uint32_t k = nbr_box[e];
            for (uint32_t p = bstart[k]; p < bstart[k + 1]; ++p, ++r) {
                uint32_t j = perm[p];
                double v[4];
                for (int d = 0; d < 3; ++d) v[d] = (pos[3 * (int64_t)j + d] + S[d]) - o[d];
                v[3] = mass[j];
                if (prec == 0) {
                    float *f = (float *)red + 4 * r;
                    for (int q = 0; q < 4; ++q) f[q] = (float)v[q];
                } else {
                    double *g = (double *)red + 4 * r;
                    for (int q = 0; q < 4; ++q) g[q] = v[q];
                }
            }
        }
    }
}

/* --------------------------------------------------------------------------------------------- */
/* a7 + a9, oracle mode (i) "redundant order": evaluate each target against its box's redundant run */
/* (records promoted to fp64); the target's local coordinate is fl_p((double)x_i - o_b) (C11).      */
/* The record that is the target itself sits in the slot-13 (self) segment at the target's offset   */
/* inside its box; it is excluded from phi and contributes exactly 0 to the field (C3).            */
/* Outputs are written in INPUT order (C12).                                                        */
/* --------------------------------------------------------------------------------------------- */
void orc_gravity_eval_redundant(int prec, int64_t B, const double *pos, double h, const double *lo,
                                const int32_t *nbox, const uint32_t *perm, const uint32_t *bkey,
                                const uint32_t *bstart, const uint32_t *nbr_off, const uint32_t *nbr_box,
                                const uint8_t *nbr_slot, const uint64_t *red_off, const void *red, double eps,
                                double *phi, double *field)
{
    int nb = orc_bits_per_dim(3, nbox);
    double eps2 = eps * eps;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t b = 0; b < B; ++b) {
        int32_t c[3];
        double o[3];
        orc_demorton(3, nb, bkey[b], c);
        box_origin(c, h, lo, o);
        /* offset of the self segment inside the run */
        uint64_t self_off = 0;
        for (uint32_t e = nbr_off[b]; e < nbr_off[b + 1]; ++e) {
            if (nbr_slot[e] == 13) break;
            self_off += bstart[nbr_box[e] + 1] - bstart[nbr_box[e]];
        }
        for (uint32_t p = bstart[b]; p < bstart[b + 1]; ++p) {
            uint32_t i = perm[p];
            double t[3];
            for (int d = 0; d < 3; ++d) {
                double v = pos[3 * (int64_t)i + d] - o[d];
                t[d] = (prec == 0) ? (double)(float)v : v;
            }
            double ph = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
            uint64_t me = red_off[b] + self_off + (p - bstart[b]);
            for (uint64_t r = red_off[b]; r < red_off[b + 1]; ++r) {
                double s[4];
                if (prec == 0)
                    for (int q = 0; q < 4; ++q) s[q] = (double)((const float *)red)[4 * r + q];
                else
                    for (int q = 0; q < 4; ++q) s[q] = ((const double *)red)[4 * r + q];
                double dx = s[0] - t[0], dy = s[1] - t[1], dz = s[2] - t[2];
                double r2 = dx * dx + dy * dy + dz * dz + eps2;
                double rinv = 1.0 / sqrt(r2);
                double mr3 = s[3] * rinv * rinv * rinv;
                if (r != me) ph -= s[3] * rinv;
                ax += mr3 * dx;
                ay += mr3 * dy;
                az += mr3 * dz;
            }
            phi[i] = ph;
            field[3 * (int64_t)i + 0] = ax;
            field[3 * (int64_t)i + 1] = ay;
            field[3 * (int64_t)i + 2] = az;
        }
    }
}

/* --------------------------------------------------------------------------------------------- */
/* a7 + a9, oracle mode (ii) "indexed order" = the plain definition: loop over the neighbour CSR and */
/* the raw records, d = (x_j + S) - x_i computed in fp64 from the (promoted) input positions.        */
/* --------------------------------------------------------------------------------------------- */
static void eval_indexed_box(int64_t b, int nb, const double *pos, const double *mass, double h,
                             const int32_t *nbox, uint32_t periodic, const uint32_t *perm, const uint32_t *bkey,
                             const uint32_t *bstart, const uint32_t *nbr_off, const uint32_t *nbr_box,
                             const uint8_t *nbr_slot, double eps2, double *phi, double *field)
{
    int32_t c[3];
    orc_demorton(3, nb, bkey[b], c);
    for (uint32_t p = bstart[b]; p < bstart[b + 1]; ++p) {
        uint32_t i = perm[p];
        const double *xi = &pos[3 * (int64_t)i];
        double ph = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
        for (uint32_t e = nbr_off[b]; e < nbr_off[b + 1]; ++e) {
            double S[3];
            slot_shift(nbr_slot[e], c, nbox, periodic, h, S);
            uint32_t k = nbr_box[e];
            for (uint32_t q = bstart[k]; q < bstart[k + 1]; ++q) {
                uint32_t j = perm[q];
                const double *xj = &pos[3 * (int64_t)j];
                double dx = (xj[0] + S[0]) - xi[0];
                double dy = (xj[1] + S[1]) - xi[1];
                double dz = (xj[2] + S[2]) - xi[2];
                double r2 = dx * dx + dy * dy + dz * dz + eps2;
                double rinv = 1.0 / sqrt(r2);
                double mr3 = mass[j] * rinv * rinv * rinv;
                if (j != i) ph -= mass[j] * rinv;
                ax += mr3 * dx;
                ay += mr3 * dy;
                az += mr3 * dz;
            }
        }
        phi[i] = ph;
        field[3 * (int64_t)i + 0] = ax;
        field[3 * (int64_t)i + 1] = ay;
        field[3 * (int64_t)i + 2] = az;
    }
}

void orc_gravity_eval_indexed(int64_t B, const double *pos, const double *mass, double h, const int32_t *nbox,
                              uint32_t periodic, const uint32_t *perm, const uint32_t *bkey,
                              const uint32_t *bstart, const uint32_t *nbr_off, const uint32_t *nbr_box,
                              const uint8_t *nbr_slot, double eps, double *phi, double *field)
{
    int nb = orc_bits_per_dim(3, nbox);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t b = 0; b < B; ++b)
        eval_indexed_box(b, nb, pos, mass, h, nbox, periodic, perm, bkey, bstart, nbr_off, nbr_box, nbr_slot,
                         eps * eps, phi, field);
}

/* The same plain definition restricted to a list of target boxes (bounded CPU-baseline samples and sampled
 * parity checks at full size); outputs of targets outside the listed boxes are left untouched. */
void orc_gravity_eval_indexed_boxes(int64_t nsel, const uint32_t *sel, const double *pos, const double *mass,
                                    double h, const int32_t *nbox, uint32_t periodic, const uint32_t *perm,
                                    const uint32_t *bkey, const uint32_t *bstart, const uint32_t *nbr_off,
                                    const uint32_t *nbr_box, const uint8_t *nbr_slot, double eps, double *phi,
                                    double *field)
{
    int nb = orc_bits_per_dim(3, nbox);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t q = 0; q < nsel; ++q)
        eval_indexed_box((int64_t)sel[q], nb, pos, mass, h, nbox, periodic, perm, bkey, bstart, nbr_off, nbr_box,
                         nbr_slot, eps * eps, phi, field);
}

/* --------------------------------------------------------------------------------------------- */
/* the paper's THREAD-level redundancy ("duplicating particle data for each     */
/* interaction pair ... an Array-of-Structures (AoS) format, where each entry contains both source   */
/* and target attributes"; S:L113-116 RedundantBuffers; partial results + reduction "through the     */
/* update process").                                                             */
/* One pair record per CSR entry e = (target box b, neighbour k, slot s), in CSR order:              */
/*   [ the n_b targets of b : fl_p(((double)x_i + 0) - o_b), m_i ]  [ the n_k sources of k, rebased  */
/*   exactly as in red (C11) ]                                                                      */
/* pr_off[e] = first record of entry e (running count of n_b + n_k); the E+1'th value = total.       */
/* --------------------------------------------------------------------------------------------- */
static void put_rec(int prec, void *buf, uint64_t r, const double *v)
{
    if (prec == 0) {
        float *f = (float *)buf + 4 * r;
        for (int q = 0; q < 4; ++q) f[q] = (float)v[q];
    } else {
        double *g = (double *)buf + 4 * r;
        for (int q = 0; q < 4; ++q) g[q] = v[q];
    }
}

static void get_rec(int prec, const void *buf, uint64_t r, double *v)
{
    if (prec == 0)
        for (int q = 0; q < 4; ++q) v[q] = (double)((const float *)buf)[4 * r + q];
    else
        for (int q = 0; q < 4; ++q) v[q] = ((const double *)buf)[4 * r + q];
}

/* offsets only (pr == NULL) or offsets + records */
void orc_gravity_pairrec(int prec, int64_t B, const double *pos, const double *mass, double h, const double *lo,
                         const int32_t *nbox, uint32_t periodic, const uint32_t *perm, const uint32_t *bkey,
                         const uint32_t *bstart, const uint32_t *nbr_off, const uint32_t *nbr_box,
                         const uint8_t *nbr_slot, uint64_t *pr_off, void *pr)
{
    int nb = orc_bits_per_dim(3, nbox);
    uint64_t r = 0;
    for (int64_t b = 0; b < B; ++b) {
        int32_t c[3];
        double o[3];
        orc_demorton(3, nb, bkey[b], c);
        box_origin(c, h, lo, o);
        for (uint32_t e = nbr_off[b]; e < nbr_off[b + 1]; ++e) {
            pr_off[e] = r;
            /* the target tuples of b */
            for (uint32_t p = bstart[b]; p < bstart[b + 1]; ++p, ++r) {
                if (!pr) continue;
                uint32_t i = perm[p];
                double v[4];
                for (int d = 0; d < 3; ++d) v[d] = (pos[3 * (int64_t)i + d] + 0.0) - o[d];
                v[3] = mass[i];
                put_rec(prec, pr, r, v);
            }
            /* the source tuples of k, with the slot's periodic image */
            double S[3];
            slot_shift(nbr_slot[e], c, nbox, periodic, h, S);
            uint32_t k = nbr_box[e];
            for (uint32_t p = bstart[k]; p < bstart[k + 1]; ++p, ++r) {
                if (!pr) continue;
                uint32_t j = perm[p];
                double v[4];
                for (int d = 0; d < 3; ++d) v[d] = (pos[3 * (int64_t)j + d] + S[d]) - o[d];
                v[3] = mass[j];
                put_rec(prec, pr, r, v);
            }
        }
    }
    pr_off[nbr_off[B]] = r;
}

/* Eval over pair records: one logical thread per (record, target) computes a partial result from the
 * record's bytes alone (the self pair -- slot 13, same sorted index -- excluded from phi, C3); then the
 * update: every target sums its partials in ascending record order (deterministic).
 * partial[4 * (slot)] = {phi, ax, ay, az}, slot = running count of targets over records (CSR order). */
void orc_gravity_eval_pairrec(int prec, int64_t B, const uint32_t *perm, const uint32_t *bstart,
                              const uint32_t *nbr_off, const uint32_t *nbr_box, const uint8_t *nbr_slot,
                              const uint64_t *pr_off, const void *pr, double eps, double *partial, double *phi,
                              double *field)
{
    double eps2 = eps * eps;
    /* partial-slot base of every box: sum over earlier boxes of |N(b)| n_b */
    uint64_t *pbase = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(B + 1));
    pbase[0] = 0;
    for (int64_t b = 0; b < B; ++b)
        pbase[b + 1] = pbase[b] + (uint64_t)(nbr_off[b + 1] - nbr_off[b]) * (bstart[b + 1] - bstart[b]);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t b = 0; b < B; ++b) {
        uint32_t nbb = bstart[b + 1] - bstart[b];
        for (uint32_t e = nbr_off[b]; e < nbr_off[b + 1]; ++e) {
            uint32_t nk = bstart[nbr_box[e] + 1] - bstart[nbr_box[e]];
            uint64_t rt = pr_off[e], rs = pr_off[e] + nbb;
            for (uint32_t j = 0; j < nbb; ++j) {
                double t[4];
                get_rec(prec, pr, rt + j, t);
                double ph = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
                for (uint32_t q = 0; q < nk; ++q) {
                    double s[4];
                    get_rec(prec, pr, rs + q, s);
                    double dx = s[0] - t[0], dy = s[1] - t[1], dz = s[2] - t[2];
                    double r2 = dx * dx + dy * dy + dz * dz + eps2;
                    double rinv = 1.0 / sqrt(r2);
                    double mr3 = s[3] * rinv * rinv * rinv;
                    if (!(nbr_slot[e] == 13 && q == j)) ph -= s[3] * rinv;
                    ax += mr3 * dx;
                    ay += mr3 * dy;
                    az += mr3 * dz;
                }
                double *o = partial + 4 * (pbase[b] + (uint64_t)(e - nbr_off[b]) * nbb + j);
                o[0] = ph;
                o[1] = ax;
                o[2] = ay;
                o[3] = az;
            }
        }
        /* update: ascending record order per target */
        for (uint32_t j = 0; j < nbb; ++j) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (uint32_t e = nbr_off[b]; e < nbr_off[b + 1]; ++e) {
                const double *o = partial + 4 * (pbase[b] + (uint64_t)(e - nbr_off[b]) * nbb + j);
                for (int q = 0; q < 4; ++q) acc[q] += o[q];
            }
            uint32_t i = perm[bstart[b] + j];
            phi[i] = acc[0];
            for (int d = 0; d < 3; ++d) field[3 * (int64_t)i + d] = acc[1 + d];
        }
    }
    free(pbase);
}

/* --------------------------------------------------------------------------------------------- */
/* Oracle mode (iii): O(N^2) brute force with the box-adjacency predicate, no lists at all.         */
/* Per dimension: periodic -> (ib_j - ib_i) mod n in {-1,0,1}; open -> |ib_j - ib_i| <= 1.  The      */
/* image is derived from the wrap: ib_j - ib_i == -(n-1) -> +L, == n-1 -> -L (needs n >= 3).         */
/* Returns -1 or the first out-of-domain index.                                                     */
/* --------------------------------------------------------------------------------------------- */
int64_t orc_gravity_brute(int64_t n, const double *pos, const double *mass, double h, const double *lo,
                          const int32_t *nbox, uint32_t periodic, double eps, double *phi, double *field)
{
    int32_t *ib = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)(n > 0 ? n : 1));
    int64_t bad = orc_bin(3, n, pos, h, lo, nbox, ib);
    if (bad >= 0) { free(ib); return bad; }
    double eps2 = eps * eps;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
        double ph = 0.0, a[3] = {0.0, 0.0, 0.0};
        for (int64_t j = 0; j < n; ++j) {
            double S[3];
            int adj = 1;
            for (int d = 0; d < 3 && adj; ++d) {
                int32_t D = ib[3 * j + d] - ib[3 * i + d];
                double L = (double)nbox[d] * h;
                S[d] = 0.0;
                if ((periodic >> d) & 1u) {
                    if (D == -(nbox[d] - 1)) S[d] = L;
                    else if (D == nbox[d] - 1) S[d] = -L;
                    else if (D < -1 || D > 1) adj = 0;
                } else if (D < -1 || D > 1) {
                    adj = 0;
                }
            }
            if (!adj) continue;
            double dx = (pos[3 * j + 0] + S[0]) - pos[3 * i + 0];
            double dy = (pos[3 * j + 1] + S[1]) - pos[3 * i + 1];
            double dz = (pos[3 * j + 2] + S[2]) - pos[3 * i + 2];
            double r2 = dx * dx + dy * dy + dz * dz + eps2;
            double rinv = 1.0 / sqrt(r2);
            double mr3 = mass[j] * rinv * rinv * rinv;
            if (j != i) ph -= mass[j] * rinv;
            a[0] += mr3 * dx;
            a[1] += mr3 * dy;
            a[2] += mr3 * dz;
        }
        phi[i] = ph;
        for (int d = 0; d < 3; ++d) field[3 * i + d] = a[d];
    }
    free(ib);
    return -1;
}

/* --------------------------------------------------------------------------------------------- */
/* Helmholtz (DBIM-like, 2D, open boundary) -- C15.                                                 */
/* G(r) = (i/4) H0^(1)(k r) = -Y0(kr)/4 + i J0(kr)/4 (glibc POSIX Bessel functions).                 */
/* Off-diagonal weight G(r) Delta^2; self cell (equal-area disk a = Delta/sqrt(pi)):                 */
/*   (i pi a / 2k) H1^(1)(k a) - 1/k^2.                                                             */
/* --------------------------------------------------------------------------------------------- */
void orc_helm_weight(double r, double delta, double k, double *re, double *im)
{
    if (r == 0.0) {
        double a = delta / sqrt(M_PI);
        double ka = k * a;
        double c = M_PI * a / (2.0 * k);
        /* i c (J1 + i Y1) - 1/k^2 = (-c Y1 - 1/k^2) + i c J1 */
        *re = -c * y1(ka) - 1.0 / (k * k);
        *im = c * j1(ka);
    } else {
        double kr = k * r;
        *re = -0.25 * y0(kr) * delta * delta;
        *im = 0.25 * j0(kr) * delta * delta;
    }
}

/* The 9t^2 pattern table: P[i][s*t + j] = weight between target sub-cell i of a box and
 * source sub-cell j of its stencil neighbour s = 3(dy+1) + (dx+1); sub-cell q = qy*st + qx (C8).
 * P is complex fp64, interleaved (re, im), [t][9t]. */
void orc_helm_table(int t, double delta, double k, double *P)
{
    int st = 0;
    while (st * st < t) ++st;
    for (int i = 0; i < t; ++i) {
        int ix = i % st, iy = i / st;
        for (int s = 0; s < 9; ++s) {
            int dx = s % 3 - 1, dy = s / 3 - 1;
            for (int j = 0; j < t; ++j) {
                int jx = j % st, jy = j / st;
                double rx = (double)(dx * st + jx - ix) * delta;
                double ry = (double)(dy * st + jy - iy) * delta;
                double re, im;
                orc_helm_weight(sqrt(rx * rx + ry * ry), delta, k, &re, &im);
                int64_t q = (int64_t)i * 9 * t + s * t + j;
                P[2 * q] = re;
                P[2 * q + 1] = im;
            }
        }
    }
}

/* Helmholtz structures (a1..a5): key = morton2(box)*t + subcell, subcell = sy*st + sx with
 * s_d = floor((x_d - o_d) / (h / st)), o_d = fma(ib_d, h, lo_d) (C8).  Every present box must hold
 * exactly one sample per sub-cell.  nbr9[9B] = box index of each stencil slot or 0xffffffff (C10).
 * Returns -1 on success, -2 if the lattice is irregular (UNSUPPORTED), else first out-of-domain. */
int64_t orc_helm_structs(int64_t n, const double *pos, double h, const double *lo, const int32_t *nbox, int t,
                         uint32_t *key, uint32_t *skey, uint32_t *perm, uint32_t *bkey, uint32_t *bstart,
                         uint32_t *nbr9, int64_t *counts)
{
    int32_t *ib = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)(n > 0 ? n : 1));
    int64_t bad = orc_bin(2, n, pos, h, lo, nbox, ib);
    if (bad >= 0) { free(ib); return bad; }
    int st = 0;
    while (st * st < t) ++st;
    double delta = h / (double)st;
    int nb = orc_bits_per_dim(2, nbox);
    for (int64_t i = 0; i < n; ++i) {
        int32_t sc[2];
        for (int d = 0; d < 2; ++d) {
            double o = fma((double)ib[2 * i + d], h, lo[d]);
            double f = floor((pos[2 * i + d] - o) / delta);
            if (!(f >= 0.0 && f < (double)st)) { free(ib); return -2; }
            sc[d] = (int32_t)f;
        }
        key[i] = orc_morton(2, nb, &ib[2 * i]) * (uint32_t)t + (uint32_t)(sc[1] * st + sc[0]);
    }
    orc_stable_sort(n, key, skey, perm);
    /* boxes = runs of key / t */
    int64_t B = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t bk = skey[i] / (uint32_t)t;
        if (i == 0 || bk != skey[i - 1] / (uint32_t)t) {
            bkey[B] = bk;
            bstart[B] = (uint32_t)i;
            ++B;
        }
        if (i > 0 && skey[i] == skey[i - 1]) { free(ib); return -2; }
    }
    bstart[B] = (uint32_t)n;
    for (int64_t b = 0; b < B; ++b)
        if (bstart[b + 1] - bstart[b] != (uint32_t)t) { free(ib); return -2; }
    for (int64_t b = 0; b < B; ++b) {
        int32_t c[2];
        orc_demorton(2, nb, bkey[b], c);
        for (int s = 0; s < 9; ++s) {
            int32_t nc[2] = {c[0] + s % 3 - 1, c[1] + s / 3 - 1};
            int64_t k = -1;
            if (nc[0] >= 0 && nc[0] < nbox[0] && nc[1] >= 0 && nc[1] < nbox[1])
                k = find_box(B, bkey, orc_morton(2, nb, nc));
            nbr9[9 * b + s] = (k < 0) ? 0xffffffffu : (uint32_t)k;
        }
    }
    counts[0] = B;
    free(ib);
    return -1;
}

/* Helmholtz a6 + a8 + a9 via the pattern table:
 *   Xg[b][s][j] = x[perm[bstart[nbr9[b][s]] + j]]  (zero segment when the neighbour is missing)
 *   y[perm[bstart[b] + i]] = sum_s sum_j P[i][s t + j] Xg[b][s][j]   (complex fp64). */
void orc_helm_eval_table(int64_t B, int t, const double *P, const double *x, const uint32_t *perm,
                         const uint32_t *bstart, const uint32_t *nbr9, double *y)
{
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < B; ++b) {
        for (int i = 0; i < t; ++i) {
            double yr = 0.0, yi = 0.0;
            for (int s = 0; s < 9; ++s) {
                uint32_t k = nbr9[9 * b + s];
                if (k == 0xffffffffu) continue; /* zero segment */
                for (int j = 0; j < t; ++j) {
                    uint32_t q = perm[bstart[k] + j];
                    const double *w = &P[2 * ((int64_t)i * 9 * t + s * t + j)];
                    double xr = x[2 * (int64_t)q], xi = x[2 * (int64_t)q + 1];
                    yr += w[0] * xr - w[1] * xi;
                    yi += w[0] * xi + w[1] * xr;
                }
            }
            uint32_t p = perm[bstart[b] + i];
            y[2 * (int64_t)p] = yr;
            y[2 * (int64_t)p + 1] = yi;
        }
    }
}

/* Helmholtz brute force: dense masked matvec straight from the positions (no table, no lists):
 * y_p = sum_q w(|x_q - x_p|) x_q over samples q whose box is adjacent to p's box (|d ib| <= 1). */
int64_t orc_helm_dense(int64_t n, const double *pos, const double *x, double h, const double *lo,
                       const int32_t *nbox, double delta, double k, double *y)
{
    int32_t *ib = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)(n > 0 ? n : 1));
    int64_t bad = orc_bin(2, n, pos, h, lo, nbox, ib);
    if (bad >= 0) { free(ib); return bad; }
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t p = 0; p < n; ++p) {
        double yr = 0.0, yi = 0.0;
        for (int64_t q = 0; q < n; ++q) {
            int32_t d0 = ib[2 * q] - ib[2 * p], d1 = ib[2 * q + 1] - ib[2 * p + 1];
            if (d0 < -1 || d0 > 1 || d1 < -1 || d1 > 1) continue;
            double rx = pos[2 * q] - pos[2 * p], ry = pos[2 * q + 1] - pos[2 * p + 1];
            double wr, wi;
            orc_helm_weight(sqrt(rx * rx + ry * ry), delta, k, &wr, &wi);
            double xr = x[2 * q], xi = x[2 * q + 1];
            yr += wr * xr - wi * xi;
            yi += wr * xi + wi * xr;
        }
        y[2 * p] = yr;
        y[2 * p + 1] = yi;
    }
    free(ib);
    return -1;
}

/* Host-thread control for the timing harness (bench.py cpu_baseline at 1 core and at all cores); no arithmetic.
 * Returns the thread count the following parallel regions use. */
#ifdef _OPENMP
#include <omp.h>
#endif
int orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}
