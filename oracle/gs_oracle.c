/* CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.
 *
 * Checker and timed CPU baseline ("port") for the B200 path; never linked by
 * the product library.  Equations follow the reference
 * (/root/reference/pkg/src/geoshoot):
 *
 *   kernels.py:121-171     G(r) and G'(r) for the conical / gaussian families,
 *                          x peak() = 1/(2 pi alpha^2) when not normalized
 *   particles.py:79-117    dq_i = sum_j G(d_ij) p_j + sigma2 p_i
 *                          dp_i = -sum_{j != i, d_ij > 0} (p_i.p_j) G'(d_ij)/d_ij (q_i - q_j)
 *                          written in the direct-difference form (the reference's
 *                          a.sum*q - a@q form cancels)
 *   particles.py:92-98     coincident interacting pair -> first (i, j), row-major
 *   particles.py:120-131   H = sum_ij (p_i.p_j) G(d_ij)
 *   integrator.py:66-121   classical RK4 with the reference's evaluation order
 *
 * cutoff > 0 selects the truncated sum over pairs with d_ij^2 < cutoff^2 (the
 * cell-list semantics, KD-1), evaluated through a uniform grid of cutoff-sized
 * cells; cutoff <= 0 is the dense all-pairs sum of the reference.
 * OpenMP parallelises over target rows.  Build: oracle/build.sh
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define GO_OK 0
#define GO_COINCIDENT 1
#define GO_NONFINITE_STAGE 2
#define GO_NONFINITE_STATE 3

typedef struct {
    int family;      /* 0 conical, 1 gaussian */
    int normalized;
    double alpha;
    double sigma2;
    double cutoff;   /* <= 0: dense */
} go_params;

static inline double kval(const go_params* k, double r) {
    double v = (k->family == 0) ? exp(-r / k->alpha) : exp(-0.5 * (r / k->alpha) * (r / k->alpha));
    if (!k->normalized) v *= 1.0 / (2.0 * M_PI * k->alpha * k->alpha);
    return v;
}

static inline double kder(const go_params* k, double r) {
    double v = (k->family == 0) ? -exp(-r / k->alpha) / k->alpha
                                : -(r / (k->alpha * k->alpha)) * exp(-0.5 * (r / k->alpha) * (r / k->alpha));
    if (!k->normalized) v *= 1.0 / (2.0 * M_PI * k->alpha * k->alpha);
    return v;
}

/* one (i, j) term; returns 1 on an interacting coincident pair */
static inline int pair_term(const go_params* k, long i, long j, const double* q, const double* p,
                            double* aq, double* ap) {
    double dx = q[2 * i] - q[2 * j], dy = q[2 * i + 1] - q[2 * j + 1];
    double r = sqrt(dx * dx + dy * dy);
    double g = kval(k, r);
    aq[0] += g * p[2 * j];
    aq[1] += g * p[2 * j + 1];
    if (j == i) return 0;
    double pdot = p[2 * i] * p[2 * j] + p[2 * i + 1] * p[2 * j + 1];
    if (r == 0.0) return pdot != 0.0;
    double a = pdot * kder(k, r) / r;
    ap[0] -= a * dx;
    ap[1] -= a * dy;
    return 0;
}

/* Cells of edge = cutoff, hashed into nb (power of two >= 2n) buckets by the bits of the double
 * cell coordinate floor(x / cutoff): no bounding box, so a flung-apart (diverging) state costs
 * the same as a compact one.  Pairs are still decided by the exact distance test.
 * The particles are counting-sorted by bucket (stable: ascending index inside a bucket) and
 * copied in that order, and targets are processed in that order, so a target's candidate
 * loads are contiguous; each target still sums bucket by bucket (stencil order dy, dx) and,
 * inside a bucket, in ascending particle index. */
typedef struct {
    double inv;
    unsigned long nb;
    long* start;   /* nb + 1 */
    long* idx;     /* n, particle indices grouped by bucket (ascending within a bucket) */
    double* qs;    /* n x 2, q in bucket order */
    double* ps;    /* n x 2, p in bucket order */
} go_grid;

static inline unsigned long long mix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static unsigned long cell_bucket(double cx, double cy, unsigned long nb) {
    double ax = cx + 0.0, ay = cy + 0.0;   /* -0.0 -> +0.0 */
    unsigned long long bx, by;
    memcpy(&bx, &ax, 8);
    memcpy(&by, &ay, 8);
    /* splitmix64 finalizer of each coordinate's bits: the low bits of small integral doubles are
     * all zero, so a plain multiply would put most cells into a few buckets */
    unsigned long long h = mix64(bx) ^ mix64(by ^ 0xC2B2AE3D27D4EB4Full);
    return (unsigned long)(h & (nb - 1));
}

static void grid_build(go_grid* g, const double* q, const double* p, long n, double cutoff) {
    g->inv = 1.0 / cutoff;
    g->nb = 1;
    while (g->nb < 2ul * (unsigned long)n) g->nb <<= 1;
    g->start = (long*)calloc(g->nb + 1, sizeof(long));
    g->idx = (long*)malloc(n * sizeof(long));
    g->qs = (double*)malloc(2 * n * sizeof(double));
    g->ps = (double*)malloc(2 * n * sizeof(double));
    unsigned long* cell = (unsigned long*)malloc(n * sizeof(unsigned long));
#pragma omp parallel for
    for (long i = 0; i < n; i++) cell[i] = cell_bucket(floor(q[2 * i] * g->inv), floor(q[2 * i + 1] * g->inv), g->nb);
    for (long i = 0; i < n; i++) g->start[cell[i] + 1]++;
    for (unsigned long c = 0; c < g->nb; c++) g->start[c + 1] += g->start[c];
    long* fill = (long*)malloc(g->nb * sizeof(long));
    memcpy(fill, g->start, g->nb * sizeof(long));
    for (long i = 0; i < n; i++) g->idx[fill[cell[i]]++] = i;
#pragma omp parallel for
    for (long s = 0; s < n; s++) {
        const long i = g->idx[s];
        g->qs[2 * s] = q[2 * i]; g->qs[2 * s + 1] = q[2 * i + 1];
        g->ps[2 * s] = p[2 * i]; g->ps[2 * s + 1] = p[2 * i + 1];
    }
    free(fill);
    free(cell);
}

static void grid_free(go_grid* g) { free(g->start); free(g->idx); free(g->qs); free(g->ps); }

/* the pair term of pair_term() on explicit values (i != j) */
static inline int pair_term_v(const go_params* k, const double* qi, const double* pi, const double* qj,
                              const double* pj, double* aq, double* ap) {
    double dx = qi[0] - qj[0], dy = qi[1] - qj[1];
    double r = sqrt(dx * dx + dy * dy);
    double g = kval(k, r);
    aq[0] += g * pj[0];
    aq[1] += g * pj[1];
    double pdot = pi[0] * pj[0] + pi[1] * pj[1];
    if (r == 0.0) return pdot != 0.0;
    double a = pdot * kder(k, r) / r;
    ap[0] -= a * dx;
    ap[1] -= a * dy;
    return 0;
}

/* rhs rows [r0, r1).  *bad = min over interacting coincident pairs of i*n + j (or -1). */
int go_rhs(const go_params* k, long n, const double* q, const double* p, double* dq, double* dp,
           long r0, long r1, long long* bad) {
    long long best = INT64_MAX;
    double c2 = k->cutoff * k->cutoff;
    if (!(k->cutoff > 0.0)) {
#pragma omp parallel for schedule(dynamic, 64) reduction(min : best)
        for (long i = r0; i < r1; i++) {
            double aq[2] = {0.0, 0.0}, ap[2] = {0.0, 0.0};
            for (long j = 0; j < n; j++) {
                if (pair_term(k, i, j, q, p, aq, ap)) {
                    long long key = (long long)i * n + j;
                    if (key < best) best = key;
                }
            }
            if (k->sigma2 != 0.0) {
                aq[0] += k->sigma2 * p[2 * i];
                aq[1] += k->sigma2 * p[2 * i + 1];
            }
            dq[2 * (i - r0)] = aq[0]; dq[2 * (i - r0) + 1] = aq[1];
            dp[2 * (i - r0)] = ap[0]; dp[2 * (i - r0) + 1] = ap[1];
        }
        *bad = (best == INT64_MAX) ? -1 : best;
        return best == INT64_MAX ? GO_OK : GO_COINCIDENT;
    }
    go_grid g;
    grid_build(&g, q, p, n, k->cutoff);
#pragma omp parallel for schedule(dynamic, 64) reduction(min : best)
    for (long t = 0; t < n; t++) {
        const long i = g.idx[t];
        if (i < r0 || i >= r1) continue;
        const double* qi = g.qs + 2 * t;
        const double* pi = g.ps + 2 * t;
        double aq[2] = {0.0, 0.0}, ap[2] = {0.0, 0.0};
        const double cx = floor(qi[0] * g.inv), cy = floor(qi[1] * g.inv);
        unsigned long seen[9];
        int ns = 0;
        for (int ddy = -1; ddy <= 1; ddy++)
            for (int ddx = -1; ddx <= 1; ddx++) {
                const unsigned long b = cell_bucket(cx + ddx, cy + ddy, g.nb);
                int dup = 0;
                for (int u = 0; u < ns; u++) dup |= seen[u] == b;
                if (dup) continue;
                seen[ns++] = b;
                for (long s = g.start[b]; s < g.start[b + 1]; s++) {
                    const double* qj = g.qs + 2 * s;
                    double dx = qi[0] - qj[0], dy = qi[1] - qj[1];
                    if (!(dx * dx + dy * dy < c2)) continue;
                    if (s == t) {  /* self pair: G(0) p_i, nothing in dp */
                        double g0 = kval(k, 0.0);
                        aq[0] += g0 * pi[0];
                        aq[1] += g0 * pi[1];
                        continue;
                    }
                    if (pair_term_v(k, qi, pi, qj, g.ps + 2 * s, aq, ap)) {
                        long long key = (long long)i * n + g.idx[s];
                        if (key < best) best = key;
                    }
                }
            }
        if (k->sigma2 != 0.0) {
            aq[0] += k->sigma2 * pi[0];
            aq[1] += k->sigma2 * pi[1];
        }
        dq[2 * (i - r0)] = aq[0]; dq[2 * (i - r0) + 1] = aq[1];
        dp[2 * (i - r0)] = ap[0]; dp[2 * (i - r0) + 1] = ap[1];
    }
    grid_free(&g);
    *bad = (best == INT64_MAX) ? -1 : best;
    return best == INT64_MAX ? GO_OK : GO_COINCIDENT;
}

double go_hamiltonian(const go_params* k, long n, const double* q, const double* p) {
    double total = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : total)
    for (long i = 0; i < n; i++) {
        double ux = 0.0, uy = 0.0;
        for (long j = 0; j < n; j++) {
            double dx = q[2 * i] - q[2 * j], dy = q[2 * i + 1] - q[2 * j + 1];
            double g = kval(k, sqrt(dx * dx + dy * dy));
            ux += g * p[2 * j];
            uy += g * p[2 * j + 1];
        }
        total += p[2 * i] * ux + p[2 * i + 1] * uy;
    }
    return total;
}

static int all_finite(const double* a, long m) {
    int ok = 1;
#pragma omp parallel for reduction(&& : ok)
    for (long i = 0; i < m; i++) ok = ok && isfinite(a[i]);
    return ok;
}

/* integrator.py:66-121.  q, p (n x 2) updated in place.  err[0] = step (1-based),
 * err[1] = i, err[2] = j of the first failure.  Returns a GO_* code. */
int go_evolve(const go_params* k, long n, double t_final, int steps, double* q, double* p, long long* err) {
    long m = 2 * n;
    double dt = t_final / steps;
    double* buf = (double*)malloc(sizeof(double) * m * 10);
    double *kq[4], *kp[4], *sq = buf + 8 * m, *sp = buf + 9 * m;
    for (int s = 0; s < 4; s++) { kq[s] = buf + 2 * s * m; kp[s] = buf + (2 * s + 1) * m; }
    int code = GO_OK;
    for (int step = 0; step < steps && code == GO_OK; step++) {
        for (int s = 0; s < 4; s++) {
            const double *qq = q, *pp = p;
            if (s > 0) {
                double c = (s == 3) ? dt : 0.5 * dt;
#pragma omp parallel for
                for (long e = 0; e < m; e++) {
                    sq[e] = q[e] + c * kq[s - 1][e];
                    sp[e] = p[e] + c * kp[s - 1][e];
                }
                if (!all_finite(sq, m) || !all_finite(sp, m)) {
                    code = GO_NONFINITE_STAGE; err[0] = step + 1; err[1] = err[2] = -1;
                    break;
                }
                qq = sq; pp = sp;
            }
            long long bad;
            if (go_rhs(k, n, qq, pp, kq[s], kp[s], 0, n, &bad) != GO_OK) {
                code = GO_COINCIDENT; err[0] = step + 1; err[1] = bad / n; err[2] = bad % n;
                break;
            }
        }
        if (code != GO_OK) break;
        double w = dt / 6.0;
#pragma omp parallel for
        for (long e = 0; e < m; e++) {
            q[e] = q[e] + w * (kq[0][e] + 2.0 * kq[1][e] + 2.0 * kq[2][e] + kq[3][e]);
            p[e] = p[e] + w * (kp[0][e] + 2.0 * kp[1][e] + 2.0 * kp[2][e] + kp[3][e]);
        }
        if (!all_finite(q, m) || !all_finite(p, m)) {
            code = GO_NONFINITE_STATE; err[0] = step + 1; err[1] = err[2] = -1;
        }
    }
    free(buf);
    return code;
}

int go_max_threads(void) { return omp_get_max_threads(); }
void go_set_threads(int t) { omp_set_num_threads(t); }
