/*
 * amber_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle for the hot path of AMBER
 * (arXiv 2601.16292): the per-step, population-wide, *synchronous* update of
 * columnar agent state (Sec. 3.1.2 lines 85-96, Sec. 3.4).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  It shares no code, header,
 * constant table or helper with the CUDA path in paper_2601_16292_b200/
 * (the two implement the same counter-based generator independently, per
 * DESIGN.md "Contract").
 *
 * Every function follows the plain definition of what it computes, one agent
 * at a time in id order, reading a step-start snapshot and writing a fresh
 * buffer.  Where the paper is silent the reading is the one in DESIGN.md
 * (section "Contract", items R1-R8, W1-W3, G1-G4, S1-S6, B1-B8, D1); each
 * function names the items it implements.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared  (no -ffast-math:
 * the Boids contract B7 requires IEEE single-rounded float ops, no FMA).
 *
 * Citation key: P:n = reference PAPER.md line n; BJ = BASELINE.json configs.
 */
#include "amber_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* R1: Philox4x32 with 10 rounds (Salmon, Moraes, Dror, Shaw, SC'11).        */
/* Round: (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1,      */
/* lo(M0*c0)); key bump (k0,k1) += (W0,W1) between rounds.                   */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R2/R3: key = (lo32(seed), hi32(seed)); counter = (lo32(b), hi32(b), t, tag). */
static void block_words(uint64_t seed, uint32_t tag, uint64_t b, uint32_t t, uint32_t w[4])
{
    uint32_t ctr[4] = {(uint32_t)b, (uint32_t)(b >> 32), t, tag};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox4x32_10(ctr, key, w);
}

/* R4: 64-bit lane u = words (2(u mod 2), 2(u mod 2)+1) of block floor(u/2), lo first. */
uint64_t orc_lane64(uint64_t seed, uint32_t tag, uint64_t u, uint32_t t)
{
    uint32_t w[4];
    block_words(seed, tag, u / 2, t, w);
    unsigned j = (unsigned)(u % 2) * 2;
    return (uint64_t)w[j] | ((uint64_t)w[j + 1] << 32);
}

/* R4: 32-bit lane u = word (u mod 4) of block floor(u/4). */
uint32_t orc_lane32(uint64_t seed, uint32_t tag, uint64_t u, uint32_t t)
{
    uint32_t w[4];
    block_words(seed, tag, u / 4, t, w);
    return w[u % 4];
}

/* R6: uniform integer in [0,n) = floor(x * n / 2^64). */
uint64_t orc_mulhi64(uint64_t x, uint64_t n)
{
    unsigned __int128 p = (unsigned __int128)x * (unsigned __int128)n;
    return (uint64_t)(p >> 64);
}

/* R7: Bernoulli(p) = [x32 < T(p)], T(p) = ceil(p * 2^32) computed in double. */
uint64_t orc_bernoulli_threshold(double p)
{
    if (!(p >= 0.0)) return 0;           /* also catches NaN */
    if (p >= 1.0) return 4294967296ull;  /* always true */
    return (uint64_t)ceil(p * 4294967296.0);
}

/* R8: uniform float in [0,1) = (x32 >> 8) * 2^-24 (exact in float32). */
float orc_u01(uint32_t x)
{
    return (float)(x >> 8) * (1.0f / 16777216.0f);
}

/* Rounding used for derived integer counts (G1 M, S1 K): floor(x + 0.5) in double. */
int64_t orc_round_count(double x)
{
    return (int64_t)floor(x + 0.5);
}

/* ------------------------------------------------------------------------ */
/* D1: order-independent, shard-additive column digest.                      */
/* digest = sum_i mix64((i << 32) ^ bits32(v_i)) mod 2^64, mix64 = the       */
/* splitmix64 finaliser.                                                     */
/* ------------------------------------------------------------------------ */
uint64_t orc_mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_digest_bits32(const uint32_t* bits, int64_t n, int64_t id0)
{
    uint64_t acc = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t id = (uint64_t)(id0 + i);
        acc += orc_mix64((id << 32) ^ (uint64_t)bits[i]);
    }
    return acc;
}

uint64_t orc_digest_u8(const uint8_t* v, int64_t n, int64_t id0)
{
    uint64_t acc = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t id = (uint64_t)(id0 + i);
        acc += orc_mix64((id << 32) ^ (uint64_t)v[i]);
    }
    return acc;
}

/* ======================================================================== */
/* Wealth transfer (Sec. 5.1.1; BJ configs 1 and 4).      */
/* ======================================================================== */

/* W1/W2: receiver of agent i at step t. */
int64_t orc_wealth_receiver(uint64_t seed, int64_t n, int64_t i, uint32_t t, int exclude_self)
{
    uint64_t x = orc_lane64(seed, ORC_TAG_WEALTH_RECV, (uint64_t)i, t);
    if (!exclude_self) return (int64_t)orc_mulhi64(x, (uint64_t)n);
    int64_t r = (int64_t)orc_mulhi64(x, (uint64_t)(n - 1));
    return r + (r >= i ? 1 : 0);
}

/*
 * W1: one synchronous step (Sec. 3.4: "all agents act on a
 * consistent state snapshot").  s_i = [w_i >= amount] read from the snapshot
 * (amount = 1 gives BJ's "wealth > 0"); every sender gives `amount` to its
 * receiver; all writes commit together.
 *   w_next_i = w_i - amount*s_i + amount * #{j : s_j = 1 and r_j = i}
 */
int orc_wealth_step(int64_t n, int32_t amount, int exclude_self, uint64_t seed, uint32_t t,
                    const int32_t* w, int32_t* w_next)
{
    if (n < 1 || amount < 1 || (exclude_self && n < 2)) return ORC_E_INVALID;
    int64_t* inc = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    if (!inc) return ORC_E_OOM;
    for (int64_t i = 0; i < n; ++i) {
        if (w[i] >= amount) {
            int64_t r = orc_wealth_receiver(seed, n, i, t, exclude_self);
            inc[r] += 1;
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = (w[i] >= amount) ? 1 : 0;
        w_next[i] = (int32_t)((int64_t)w[i] - amount * s + amount * inc[i]);
    }
    free(inc);
    return 0;
}

/*
 * Runs `steps` steps starting at step index t0; `w` is updated in place.
 * After each step k it records (if the pointers are non-NULL) the step's
 * observables (SPEC run_model: collect after step): total wealth, the number
 * of agents with w > 0, and the D1 digest of the wealth column.
 */
int orc_wealth_run(int64_t n, int32_t amount, int exclude_self, uint64_t seed, uint32_t t0,
                   int64_t steps, int32_t* w, int64_t* total_out, int64_t* active_out,
                   uint64_t* digest_out)
{
    int32_t* tmp = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (!tmp) return ORC_E_OOM;
    for (int64_t k = 0; k < steps; ++k) {
        int rc = orc_wealth_step(n, amount, exclude_self, seed, t0 + (uint32_t)k, w, tmp);
        if (rc) { free(tmp); return rc; }
        memcpy(w, tmp, (size_t)n * sizeof(int32_t));
        if (total_out || active_out) {
            int64_t tot = 0, act = 0;
            for (int64_t i = 0; i < n; ++i) { tot += w[i]; act += (w[i] > 0); }
            if (total_out) total_out[k] = tot;
            if (active_out) active_out[k] = act;
        }
        if (digest_out) digest_out[k] = orc_digest_bits32((const uint32_t*)w, n, 0);
    }
    free(tmp);
    return 0;
}

/* ======================================================================== */
/* Erdos-Renyi contact graph G(n, M) as undirected CSR (Sec. 4.1   */
/* line 177; BJ configs 2 and 5).  Items G1-G3.                              */
/* ======================================================================== */

static int cmp_u64(const void* a, const void* b)
{
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return (x > y) - (x < y);
}

static int cmp_i32(const void* a, const void* b)
{
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* G2: endpoints of draw e. */
void orc_er_draw(uint64_t seed, int64_t n, int64_t e, int64_t* u_out, int64_t* v_out)
{
    uint64_t xu = orc_lane64(seed, ORC_TAG_GRAPH, 2 * (uint64_t)e, 0);
    uint64_t xv = orc_lane64(seed, ORC_TAG_GRAPH, 2 * (uint64_t)e + 1, 0);
    int64_t u = (int64_t)orc_mulhi64(xu, (uint64_t)n);
    int64_t vp = (int64_t)orc_mulhi64(xv, (uint64_t)(n - 1));
    *u_out = u;
    *v_out = vp + (vp >= u ? 1 : 0);
}

/*
 * G1-G3: M draws, canonical (min,max) pairs, sorted and de-duplicated, both
 * arc directions in CSR with ascending neighbour lists.  row_ptr has n+1
 * entries; col needs capacity 2*m.  Returns M' (unique edges) or < 0.
 */
int64_t orc_er_graph(int64_t n, int64_t m, uint64_t seed, int32_t* row_ptr, int32_t* col)
{
    if (n < 2 || m < 0 || n > 2147483647) return ORC_E_INVALID;
    uint64_t* keys = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
    if (!keys) return ORC_E_OOM;
    for (int64_t e = 0; e < m; ++e) {
        int64_t u, v;
        orc_er_draw(seed, n, e, &u, &v);
        uint64_t a = (uint64_t)(u < v ? u : v), b = (uint64_t)(u < v ? v : u);
        keys[e] = (a << 32) | b;
    }
    qsort(keys, (size_t)m, sizeof(uint64_t), cmp_u64);
    int64_t mu = 0;
    for (int64_t e = 0; e < m; ++e)
        if (e == 0 || keys[e] != keys[e - 1]) keys[mu++] = keys[e];
    if (2 * mu > 2147483647) { free(keys); return ORC_E_INVALID; }

    int64_t* deg = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    if (!deg) { free(keys); return ORC_E_OOM; }
    for (int64_t e = 0; e < mu; ++e) {
        deg[keys[e] >> 32] += 1;
        deg[keys[e] & 0xFFFFFFFFull] += 1;
    }
    row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + (int32_t)deg[i];
    for (int64_t i = 0; i < n; ++i) deg[i] = row_ptr[i]; /* fill cursor */
    for (int64_t e = 0; e < mu; ++e) {
        int64_t a = (int64_t)(keys[e] >> 32), b = (int64_t)(keys[e] & 0xFFFFFFFFull);
        col[deg[a]++] = (int32_t)b;
        col[deg[b]++] = (int32_t)a;
    }
    for (int64_t i = 0; i < n; ++i)
        qsort(col + row_ptr[i], (size_t)(row_ptr[i + 1] - row_ptr[i]), sizeof(int32_t), cmp_i32);
    free(deg);
    free(keys);
    return mu;
}

/* ======================================================================== */
/* SIR on a contact graph (Sec. 5.1.1, Listing 2 lines    */
/* 134-145; BJ configs 2 and 5).  Items S1-S6.                               */
/* ======================================================================== */

typedef struct { uint64_t key; int64_t id; } key_id;

static int cmp_key_id(const void* a, const void* b)
{
    const key_id* x = (const key_id*)a;
    const key_id* y = (const key_id*)b;
    if (x->key != y->key) return (x->key > y->key) - (x->key < y->key);
    return (x->id > y->id) - (x->id < y->id);
}

/* S1: the k agents with the smallest (lane64(SIR_INIT, i, 0), i) start I. */
int orc_sir_init(int64_t n, int64_t k, uint64_t seed, uint8_t* state)
{
    if (n < 1 || k < 0 || k > n) return ORC_E_INVALID;
    key_id* ki = (key_id*)malloc((size_t)n * sizeof(key_id));
    if (!ki) return ORC_E_OOM;
    for (int64_t i = 0; i < n; ++i) {
        ki[i].key = orc_lane64(seed, ORC_TAG_SIR_INIT, (uint64_t)i, 0);
        ki[i].id = i;
    }
    qsort(ki, (size_t)n, sizeof(key_id), cmp_key_id);
    for (int64_t i = 0; i < n; ++i) state[i] = ORC_S;
    for (int64_t r = 0; r < k; ++r) state[ki[r].id] = ORC_I;
    free(ki);
    return 0;
}

/* S2/S3: transmission draw on the undirected edge {a, b} at step t. */
uint32_t orc_sir_tx_word(uint64_t seed, int64_t a, int64_t b, uint32_t t)
{
    int64_t lo = a < b ? a : b, hi = a < b ? b : a;
    uint32_t ctr[4] = {(uint32_t)lo, (uint32_t)hi, t, ORC_TAG_SIR_TX};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t w[4];
    orc_philox4x32_10(ctr, key, w);
    return w[0];
}

/*
 * S2: one synchronous step from snapshot x into x_next.
 *  - S agent s becomes I iff some neighbour i has x[i] = I and the edge draw
 *    on {s, i} at step t is below T(beta)  (per-edge reading of Listing 2's
 *    "contact with infected neighbors", BJ config 2);
 *  - I agent becomes R iff lane32(SIR_REC, i, t) < T(gamma);
 *  - R stays R.  Both transitions commit together.
 */
void orc_sir_step(int64_t n, const int32_t* row_ptr, const int32_t* col, uint64_t seed,
                  uint32_t t, uint64_t t_beta, uint64_t t_gamma, const uint8_t* x,
                  uint8_t* x_next)
{
    for (int64_t s = 0; s < n; ++s) {
        if (x[s] == ORC_S) {
            int infected = 0;
            for (int32_t p = row_ptr[s]; p < row_ptr[s + 1]; ++p) {
                int64_t i = col[p];
                if (x[i] == ORC_I && (uint64_t)orc_sir_tx_word(seed, s, i, t) < t_beta) {
                    infected = 1;
                    break;
                }
            }
            x_next[s] = infected ? ORC_I : ORC_S;
        } else if (x[s] == ORC_I) {
            uint32_t d = orc_lane32(seed, ORC_TAG_SIR_REC, (uint64_t)s, t);
            x_next[s] = ((uint64_t)d < t_gamma) ? ORC_R : ORC_I;
        } else {
            x_next[s] = ORC_R;
        }
    }
}

/* Runs `steps` steps from step index t0, state updated in place; after each
 * step records S, I, R counts (counts_out[3k..3k+2]) and the D1 digest. */
int orc_sir_run(int64_t n, const int32_t* row_ptr, const int32_t* col, uint64_t seed,
                double beta, double gamma, uint32_t t0, int64_t steps, uint8_t* state,
                int64_t* counts_out, uint64_t* digest_out)
{
    uint8_t* tmp = (uint8_t*)malloc((size_t)n);
    if (!tmp) return ORC_E_OOM;
    uint64_t tb = orc_bernoulli_threshold(beta), tg = orc_bernoulli_threshold(gamma);
    for (int64_t k = 0; k < steps; ++k) {
        orc_sir_step(n, row_ptr, col, seed, t0 + (uint32_t)k, tb, tg, state, tmp);
        memcpy(state, tmp, (size_t)n);
        if (counts_out) {
            int64_t c[3] = {0, 0, 0};
            for (int64_t i = 0; i < n; ++i) c[state[i]] += 1;
            counts_out[3 * k + 0] = c[0];
            counts_out[3 * k + 1] = c[1];
            counts_out[3 * k + 2] = c[2];
        }
        if (digest_out) digest_out[k] = orc_digest_u8(state, n, 0);
    }
    free(tmp);
    return 0;
}

/*
 * One sweep replicate end to end (S6; Sec. 4.2 "configurable
 * replication counts"): own G(n, M) graph from its seed, K initial infected,
 * `steps` steps; returns final R count (R fraction = R / n).
 */
int64_t orc_sir_replicate(int64_t n, double mean_degree, double beta, double gamma,
                          double init_frac, uint64_t seed, int64_t steps)
{
    int64_t m = orc_round_count((double)n * mean_degree / 2.0);
    int64_t k = orc_round_count(init_frac * (double)n);
    int32_t* row_ptr = (int32_t*)malloc((size_t)(n + 1) * sizeof(int32_t));
    int32_t* col = (int32_t*)malloc((size_t)(2 * m > 0 ? 2 * m : 1) * sizeof(int32_t));
    uint8_t* st = (uint8_t*)malloc((size_t)n);
    if (!row_ptr || !col || !st) { free(row_ptr); free(col); free(st); return ORC_E_OOM; }
    int64_t rc = orc_er_graph(n, m, seed, row_ptr, col);
    if (rc >= 0) rc = orc_sir_init(n, k, seed, st);
    if (rc >= 0) rc = orc_sir_run(n, row_ptr, col, seed, beta, gamma, 0, steps, st, NULL, NULL);
    int64_t r = 0;
    if (rc >= 0)
        for (int64_t i = 0; i < n; ++i) r += (st[i] == ORC_R);
    free(row_ptr); free(col); free(st);
    return rc < 0 ? rc : r;
}

/* S5/S6: final R fraction per replicate (exact ratio of integers). */
int orc_sir_sweep(int64_t n, double mean_degree, double gamma, double init_frac,
                  int64_t n_reps, const double* betas, const uint64_t* seeds, int64_t steps,
                  double* out_final_r_frac)
{
    for (int64_t r = 0; r < n_reps; ++r) {
        int64_t rr = orc_sir_replicate(n, mean_degree, betas[r], gamma, init_frac, seeds[r], steps);
        if (rr < 0) return (int)rr;
        out_final_r_frac[r] = (double)rr / (double)n;
    }
    return 0;
}

/* ======================================================================== */
/* Boids flocking in a periodic box (BJ config 3; continuous space per       */
/* PAPER.md Sec. 4.1, wrapped boundary).  Items B1-B7.              */
/* ======================================================================== */

/* B1: initial positions and unit velocities. */
void orc_boids_init(int64_t n, float L, uint64_t seed, float* px, float* py, float* vx, float* vy)
{
    for (int64_t i = 0; i < n; ++i) {
        px[i] = L * orc_u01(orc_lane32(seed, ORC_TAG_BOIDS_POS, 2 * (uint64_t)i, 0));
        py[i] = L * orc_u01(orc_lane32(seed, ORC_TAG_BOIDS_POS, 2 * (uint64_t)i + 1, 0));
        /* rejection sampling of a direction in the unit disc (no sin/cos) */
        for (uint32_t attempt = 0;; ++attempt) {
            uint32_t w[4];
            uint32_t ctr[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), attempt,
                               ORC_TAG_BOIDS_VEL};
            uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
            orc_philox4x32_10(ctr, key, w);
            float a = 2.0f * orc_u01(w[0]) - 1.0f;
            float b = 2.0f * orc_u01(w[1]) - 1.0f;
            float s2 = a * a + b * b;
            if (s2 > 0.0f && s2 <= 1.0f) {
                float s = sqrtf(s2);
                vx[i] = a / s;
                vy[i] = b / s;
                break;
            }
        }
    }
}

/* B3: fixed-point quantisation Q(f) = round-half-even(f * 2^24). */
static int64_t q24(float f)
{
    return (int64_t)llrintf(f * 16777216.0f);
}

/* B2: minimum-image displacement component. */
static float min_image(float d, float L, float halfL)
{
    if (d > halfL) d -= L;
    else if (d < -halfL) d += L;
    return d;
}

typedef struct {
    int64_t n, sdx, sdy, svx, svy, ssx, ssy;
} boid_acc;

/* B2/B3: accumulate candidate j into agent i's neighbour sums. */
static void boid_consider(const orc_boids_params* P, float xi, float yi, float xj, float yj,
                          float vxj, float vyj, boid_acc* a)
{
    float halfL = 0.5f * P->L;
    float dx = min_image(xj - xi, P->L, halfL);
    float dy = min_image(yj - yi, P->L, halfL);
    float d2 = dx * dx + dy * dy;
    if (d2 <= P->R * P->R) {
        a->n += 1;
        a->sdx += q24(dx); a->sdy += q24(dy);
        a->svx += q24(vxj); a->svy += q24(vyj);
        if (d2 <= P->rs * P->rs) { a->ssx += q24(dx); a->ssy += q24(dy); }
    }
}

/* B4-B6: rules, speed clamp, integrate, wrap. */
static void boid_update(const orc_boids_params* P, float xi, float yi, float vxi, float vyi,
                        const boid_acc* a, float* nx, float* ny, float* nvx, float* nvy)
{
    float ux = vxi, uy = vyi;
    if (a->n > 0) {
        double nd = (double)a->n;
        float cohx = (float)(((double)a->sdx / 16777216.0) / nd);
        float cohy = (float)(((double)a->sdy / 16777216.0) / nd);
        float avx = (float)(((double)a->svx / 16777216.0) / nd);
        float avy = (float)(((double)a->svy / 16777216.0) / nd);
        float sepx = (float)((double)a->ssx / 16777216.0);
        float sepy = (float)((double)a->ssy / 16777216.0);
        ux = ((vxi + P->wc * cohx) + P->wa * (avx - vxi)) - P->ws * sepx;
        uy = ((vyi + P->wc * cohy) + P->wa * (avy - vyi)) - P->ws * sepy;
    }
    float s2 = ux * ux + uy * uy;
    if (s2 > P->vmax * P->vmax) {
        float f = P->vmax / sqrtf(s2);
        ux = ux * f;
        uy = uy * f;
    }
    float x = xi + ux * P->dt;
    float y = yi + uy * P->dt;
    if (x < 0.0f) x += P->L;
    if (x >= P->L) x -= P->L;
    if (y < 0.0f) y += P->L;
    if (y >= P->L) y -= P->L;
    *nx = x; *ny = y; *nvx = ux; *nvy = uy;
}

/* The plain definition: every agent scans every other agent (O(N^2)). */
void orc_boids_step_brute(int64_t n, const orc_boids_params* P, const float* px, const float* py,
                          const float* vx, const float* vy, float* opx, float* opy, float* ovx,
                          float* ovy)
{
    for (int64_t i = 0; i < n; ++i) {
        boid_acc a = {0, 0, 0, 0, 0, 0, 0};
        for (int64_t j = 0; j < n; ++j)
            if (j != i) boid_consider(P, px[i], py[i], px[j], py[j], vx[j], vy[j], &a);
        boid_update(P, px[i], py[i], vx[i], vy[i], &a, &opx[i], &opy[i], &ovx[i], &ovy[i]);
    }
}

/* Brute force for a list of agents only (sampled outputs at full N). */
void orc_boids_step_brute_sample(int64_t n, const orc_boids_params* P, const float* px,
                                 const float* py, const float* vx, const float* vy,
                                 int64_t n_sample, const int64_t* ids, float* opx, float* opy,
                                 float* ovx, float* ovy, int64_t* n_neigh)
{
    for (int64_t s = 0; s < n_sample; ++s) {
        int64_t i = ids[s];
        boid_acc a = {0, 0, 0, 0, 0, 0, 0};
        for (int64_t j = 0; j < n; ++j)
            if (j != i) boid_consider(P, px[i], py[i], px[j], py[j], vx[j], vy[j], &a);
        boid_update(P, px[i], py[i], vx[i], vy[i], &a, &opx[s], &opy[s], &ovx[s], &ovy[s]);
        if (n_neigh) n_neigh[s] = a.n;
    }
}

/* Cell count per side for the oracle's own cell list: cells of side >= R
 * with a 0.1% margin so float rounding of the cell index can never hide a
 * neighbour outside the 3x3 stencil.  Returns 0 when the box is too small
 * for a distinct 3x3 stencil (the binned step then falls back to brute). */
static int64_t oracle_cells_per_side(const orc_boids_params* P)
{
    double nc = floor((double)P->L / ((double)P->R * 1.001));
    if (nc < 3.0) return 0;
    if (nc > 4096.0) nc = 4096.0;
    return (int64_t)nc;
}

/*
 * Same rule as orc_boids_step_brute, candidates taken from the 3x3 block of
 * uniform cells around each agent (a cell list: the plain accelerator for a
 * fixed-radius query).  Because the sums are exact integers (B3) the result
 * equals the brute-force step bit for bit; tests pin that.
 */
int orc_boids_step_binned(int64_t n, const orc_boids_params* P, const float* px, const float* py,
                          const float* vx, const float* vy, float* opx, float* opy, float* ovx,
                          float* ovy)
{
    int64_t nc = oracle_cells_per_side(P);
    if (nc == 0) {
        orc_boids_step_brute(n, P, px, py, vx, vy, opx, opy, ovx, ovy);
        return 0;
    }
    int64_t ncell = nc * nc;
    int64_t* start = (int64_t*)calloc((size_t)(ncell + 1), sizeof(int64_t));
    int64_t* cell_of = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t* cur = (int64_t*)malloc((size_t)(ncell + 1) * sizeof(int64_t));
    if (!start || !cell_of || !order || !cur) {
        free(start); free(cell_of); free(order); free(cur);
        return ORC_E_OOM;
    }
    double scale = (double)nc / (double)P->L;
    for (int64_t i = 0; i < n; ++i) {
        int64_t cx = (int64_t)((double)px[i] * scale), cy = (int64_t)((double)py[i] * scale);
        if (cx >= nc) cx = nc - 1;
        if (cy >= nc) cy = nc - 1;
        if (cx < 0) cx = 0;
        if (cy < 0) cy = 0;
        cell_of[i] = cy * nc + cx;
        start[cell_of[i] + 1] += 1;
    }
    for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
    memcpy(cur, start, (size_t)(ncell + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) order[cur[cell_of[i]]++] = i;

    for (int64_t i = 0; i < n; ++i) {
        boid_acc a = {0, 0, 0, 0, 0, 0, 0};
        int64_t cx = cell_of[i] % nc, cy = cell_of[i] / nc;
        for (int64_t dy = -1; dy <= 1; ++dy)
            for (int64_t dx = -1; dx <= 1; ++dx) {
                int64_t c = ((cy + dy + nc) % nc) * nc + ((cx + dx + nc) % nc);
                for (int64_t p = start[c]; p < start[c + 1]; ++p) {
                    int64_t j = order[p];
                    if (j != i) boid_consider(P, px[i], py[i], px[j], py[j], vx[j], vy[j], &a);
                }
            }
        boid_update(P, px[i], py[i], vx[i], vy[i], &a, &opx[i], &opy[i], &ovx[i], &ovy[i]);
    }
    free(start); free(cell_of); free(order); free(cur);
    return 0;
}

/* Per-step observables (B8), accumulated in double in id order. */
void orc_boids_metrics(int64_t n, const float* vx, const float* vy, double* mean_speed,
                       double* polarisation)
{
    double ss = 0.0, ux = 0.0, uy = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double a = (double)vx[i], b = (double)vy[i];
        double sp = sqrt(a * a + b * b);
        ss += sp;
        if (sp > 0.0) { ux += a / sp; uy += b / sp; }
    }
    *mean_speed = n > 0 ? ss / (double)n : 0.0;
    *polarisation = n > 0 ? sqrt(ux * ux + uy * uy) / (double)n : 0.0;
}

/* Runs `steps` binned steps in place, recording mean speed / polarisation. */
int orc_boids_run(int64_t n, const orc_boids_params* P, int64_t steps, float* px, float* py,
                  float* vx, float* vy, double* mean_speed_out, double* polar_out)
{
    size_t bytes = (size_t)(n > 0 ? n : 1) * sizeof(float);
    float* t0 = (float*)malloc(bytes);
    float* t1 = (float*)malloc(bytes);
    float* t2 = (float*)malloc(bytes);
    float* t3 = (float*)malloc(bytes);
    if (!t0 || !t1 || !t2 || !t3) { free(t0); free(t1); free(t2); free(t3); return ORC_E_OOM; }
    for (int64_t k = 0; k < steps; ++k) {
        int rc = orc_boids_step_binned(n, P, px, py, vx, vy, t0, t1, t2, t3);
        if (rc) { free(t0); free(t1); free(t2); free(t3); return rc; }
        memcpy(px, t0, (size_t)n * sizeof(float));
        memcpy(py, t1, (size_t)n * sizeof(float));
        memcpy(vx, t2, (size_t)n * sizeof(float));
        memcpy(vy, t3, (size_t)n * sizeof(float));
        if (mean_speed_out || polar_out) {
            double ms, po;
            orc_boids_metrics(n, vx, vy, &ms, &po);
            if (mean_speed_out) mean_speed_out[k] = ms;
            if (polar_out) polar_out[k] = po;
        }
    }
    free(t0); free(t1); free(t2); free(t3);
    return 0;
}

/*
 * B pin (vi): the same rules in double-precision real-number-like arithmetic
 * (no fixed point, no float rounding of intermediate steps).  Used only to
 * check that the float32 contract stays within the one-step tolerance of the
 * plain definition.  Positions/velocities in and out are doubles.
 */
void orc_boids_step_brute_f64(int64_t n, const orc_boids_params* P, const double* px,
                              const double* py, const double* vx, const double* vy, double* opx,
                              double* opy, double* ovx, double* ovy)
{
    double L = P->L, halfL = 0.5 * L, R2 = (double)P->R * P->R, rs2 = (double)P->rs * P->rs;
    for (int64_t i = 0; i < n; ++i) {
        double cnt = 0, sdx = 0, sdy = 0, svx = 0, svy = 0, ssx = 0, ssy = 0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double dx = px[j] - px[i], dy = py[j] - py[i];
            if (dx > halfL) dx -= L; else if (dx < -halfL) dx += L;
            if (dy > halfL) dy -= L; else if (dy < -halfL) dy += L;
            double d2 = dx * dx + dy * dy;
            if (d2 <= R2) {
                cnt += 1; sdx += dx; sdy += dy; svx += vx[j]; svy += vy[j];
                if (d2 <= rs2) { ssx += dx; ssy += dy; }
            }
        }
        double ux = vx[i], uy = vy[i];
        if (cnt > 0) {
            ux = vx[i] + P->wc * (sdx / cnt) + P->wa * (svx / cnt - vx[i]) - P->ws * ssx;
            uy = vy[i] + P->wc * (sdy / cnt) + P->wa * (svy / cnt - vy[i]) - P->ws * ssy;
        }
        double s2 = ux * ux + uy * uy, vm = P->vmax;
        if (s2 > vm * vm) { double f = vm / sqrt(s2); ux *= f; uy *= f; }
        double x = px[i] + ux * P->dt, y = py[i] + uy * P->dt;
        if (x < 0) x += L;
        if (x >= L) x -= L;
        if (y < 0) y += L;
        if (y >= L) y -= L;
        opx[i] = x; opy[i] = y; ovx[i] = ux; ovy[i] = uy;
    }
}

/* ======================================================================== */
/* Random Walk (Sec. 5.1.1: "agents move in continuous 2D */
/* space according to random velocity vectors with boundary handling";      */
/* Sec. 5.3: "vector additions ... boundary handling applied as    */
/* vectorized clipping").  Contract items K1-K3.                */
/* ======================================================================== */

/* K1: positions uniform in [0, L)^2 from 32-bit lanes 2i, 2i+1 of tag 0x30. */
void orc_walk_init(int64_t n, float L, uint64_t seed, float* px, float* py)
{
    for (int64_t i = 0; i < n; ++i) {
        px[i] = L * orc_u01(orc_lane32(seed, ORC_TAG_WALK_POS, 2 * (uint64_t)i, 0));
        py[i] = L * orc_u01(orc_lane32(seed, ORC_TAG_WALK_POS, 2 * (uint64_t)i + 1, 0));
    }
}

/* K2/K3: v = (2u - 1) * vmax per component (u from lanes 2i, 2i+1 of tag 0x31
 * at step t); p' = clip(p + v) into [0, L - ulp] (the largest float below L:
 * the half-open box of SPEC's bounded space). */
void orc_walk_step(int64_t n, float L, float vmax, uint64_t seed, uint32_t t, const float* px, const float* py,
                   float* opx, float* opy)
{
    const float hi = nextafterf(L, 0.0f);
    for (int64_t i = 0; i < n; ++i) {
        float vx = (2.0f * orc_u01(orc_lane32(seed, ORC_TAG_WALK_VEL, 2 * (uint64_t)i, t)) - 1.0f) * vmax;
        float vy = (2.0f * orc_u01(orc_lane32(seed, ORC_TAG_WALK_VEL, 2 * (uint64_t)i + 1, t)) - 1.0f) * vmax;
        float x = px[i] + vx, y = py[i] + vy;
        if (x < 0.0f) x = 0.0f;
        if (x > hi) x = hi;
        if (y < 0.0f) y = 0.0f;
        if (y > hi) y = hi;
        opx[i] = x;
        opy[i] = y;
    }
}

/* Runs `steps` steps in place; records the mean displacement from the origin
 * positions (ox, oy) after each step (SPEC run_walk metric), in double. */
int orc_walk_run(int64_t n, float L, float vmax, uint64_t seed, uint32_t t0, int64_t steps, float* px, float* py,
                 const float* ox, const float* oy, double* mean_disp_out)
{
    size_t bytes = (size_t)(n > 0 ? n : 1) * sizeof(float);
    float* tx = (float*)malloc(bytes);
    float* ty = (float*)malloc(bytes);
    if (!tx || !ty) { free(tx); free(ty); return ORC_E_OOM; }
    for (int64_t k = 0; k < steps; ++k) {
        orc_walk_step(n, L, vmax, seed, t0 + (uint32_t)k, px, py, tx, ty);
        memcpy(px, tx, (size_t)n * sizeof(float));
        memcpy(py, ty, (size_t)n * sizeof(float));
        if (mean_disp_out) {
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) {
                double dx = (double)px[i] - (double)ox[i], dy = (double)py[i] - (double)oy[i];
                s += sqrt(dx * dx + dy * dy);
            }
            mean_disp_out[k] = n > 0 ? s / (double)n : 0.0;
        }
    }
    free(tx); free(ty);
    return 0;
}

/* ======================================================================== */
/* SIR in continuous space -- the paper's SIR benchmark (PAPER.md Sec.      */
/* 5.1.1 line 203: "agents in continuous 2D space ... based on contact with */
/* infected neighbors within a fixed radius"; Listing 2: one  */
/* draw per susceptible with >= 1 infected neighbour).  Items C1-C4.        */
/* ======================================================================== */

/* C1: static positions uniform in [0, L)^2 (lanes 2i, 2i+1 of tag 0x40) and
 * the K agents with the smallest (lane64(0x42, i, 0), i) infected (as S1). */
int orc_sirs_init(int64_t n, float L, int64_t k, uint64_t seed, float* px, float* py, uint8_t* state)
{
    for (int64_t i = 0; i < n; ++i) {
        px[i] = L * orc_u01(orc_lane32(seed, ORC_TAG_SIRS_POS, 2 * (uint64_t)i, 0));
        py[i] = L * orc_u01(orc_lane32(seed, ORC_TAG_SIRS_POS, 2 * (uint64_t)i + 1, 0));
    }
    if (n < 1 || k < 0 || k > n) return ORC_E_INVALID;
    key_id* ki = (key_id*)malloc((size_t)n * sizeof(key_id));
    if (!ki) return ORC_E_OOM;
    for (int64_t i = 0; i < n; ++i) {
        ki[i].key = orc_lane64(seed, ORC_TAG_SIRS_INIT, (uint64_t)i, 0);
        ki[i].id = i;
    }
    qsort(ki, (size_t)n, sizeof(key_id), cmp_key_id);
    for (int64_t i = 0; i < n; ++i) state[i] = ORC_S;
    for (int64_t j = 0; j < k; ++j) state[ki[j].id] = ORC_I;
    free(ki);
    return 0;
}

/* C2: contact lists by brute force: j != i with dx*dx + dy*dy <= r*r (float,
 * bounded box, no wrap; boundary inclusive as SPEC neighbors_within), rows
 * ascending.  Returns the number of arcs (or < 0; ORC_E_INVALID if > cap). */
int64_t orc_sirs_contacts(int64_t n, const float* px, const float* py, float r, int32_t* row_ptr, int32_t* col,
                          int64_t cap)
{
    const float r2 = r * r;
    int64_t a = 0;
    row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            float dx = px[j] - px[i], dy = py[j] - py[i];
            if (dx * dx + dy * dy <= r2) {
                if (a >= cap) return ORC_E_INVALID;
                col[a++] = (int32_t)j;
            }
        }
        row_ptr[i + 1] = (int32_t)a;
    }
    return a;
}

/* C2 at scale: the same contact lists as orc_sirs_contacts (same float test,
 * same ascending rows) found through a uniform grid instead of all pairs:
 * nc = max(1, floor(L / (1.001 r))) cells per side of width L / nc >= r, so
 * every pair within r lies in the same or an adjacent (clipped, no wrap)
 * cell.  Plain counting sort of the agents by cell, then per agent the 3x3
 * clipped stencil, the float test, and a sort of the row.  Pinned against
 * orc_sirs_contacts (brute force) in tests/test_oracle_sirs.py. */
int64_t orc_sirs_contacts_grid(int64_t n, const float* px, const float* py, float L, float r, int32_t* row_ptr,
                               int32_t* col, int64_t cap)
{
    const float r2 = r * r;
    int64_t nc = (int64_t)floor((double)L / (1.001 * (double)r));
    if (nc < 1) nc = 1;
    if (nc > 65536) nc = 65536;
    const double cs = (double)L / (double)nc;
    int64_t ncell = nc * nc;
    int64_t* start = (int64_t*)calloc((size_t)ncell + 1, sizeof(int64_t));
    int64_t* cell = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int32_t* list = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    int32_t* row = NULL;
    int64_t row_cap = 0;
    if (!start || !cell || !list) { free(start); free(cell); free(list); return ORC_E_OOM; }
    for (int64_t i = 0; i < n; ++i) {
        int64_t cx = (int64_t)((double)px[i] / cs), cy = (int64_t)((double)py[i] / cs);
        if (cx < 0) cx = 0;
        if (cx >= nc) cx = nc - 1;
        if (cy < 0) cy = 0;
        if (cy >= nc) cy = nc - 1;
        cell[i] = cy * nc + cx;
        start[cell[i] + 1] += 1;
    }
    for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
    {
        int64_t* fill = (int64_t*)malloc((size_t)ncell * sizeof(int64_t));
        if (!fill) { free(start); free(cell); free(list); return ORC_E_OOM; }
        memcpy(fill, start, (size_t)ncell * sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) list[fill[cell[i]]++] = (int32_t)i;  /* id order within a cell */
        free(fill);
    }
    /* cell-ordered copies of the positions (the same float values) */
    float* sx = (float*)malloc((size_t)(n > 0 ? n : 1) * sizeof(float));
    float* sy = (float*)malloc((size_t)(n > 0 ? n : 1) * sizeof(float));
    if (!sx || !sy) { free(sx); free(sy); free(start); free(cell); free(list); return ORC_E_OOM; }
    for (int64_t q = 0; q < n; ++q) { sx[q] = px[list[q]]; sy[q] = py[list[q]]; }
    int64_t a = 0;
    row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t cx = cell[i] % nc, cy = cell[i] / nc, k = 0;
        for (int64_t y = cy - 1; y <= cy + 1; ++y) {
            if (y < 0 || y >= nc) continue;
            for (int64_t x = cx - 1; x <= cx + 1; ++x) {
                if (x < 0 || x >= nc) continue;
                int64_t c = y * nc + x;
                for (int64_t q = start[c]; q < start[c + 1]; ++q) {
                    int64_t j = list[q];
                    if (j == i) continue;
                    float dx = sx[q] - px[i], dy = sy[q] - py[i];
                    if (dx * dx + dy * dy <= r2) {
                        if (k >= row_cap) {
                            row_cap = row_cap ? 2 * row_cap : 64;
                            int32_t* nr = (int32_t*)realloc(row, (size_t)row_cap * sizeof(int32_t));
                            if (!nr) { free(row); free(sx); free(sy); free(start); free(cell); free(list); return ORC_E_OOM; }
                            row = nr;
                        }
                        row[k++] = (int32_t)j;
                    }
                }
            }
        }
        qsort(row, (size_t)k, sizeof(int32_t), cmp_i32);
        if (a + k > cap) { free(row); free(sx); free(sy); free(start); free(cell); free(list); return ORC_E_INVALID; }
        memcpy(col + a, row, (size_t)k * sizeof(int32_t));
        a += k;
        if (a > 2147483647) { free(row); free(sx); free(sy); free(start); free(cell); free(list); return ORC_E_INVALID; }
        row_ptr[i + 1] = (int32_t)a;
    }
    free(row); free(sx); free(sy); free(start); free(cell); free(list);
    return a;
}

/* C3: one synchronous step: a susceptible with at least one infected contact
 * takes ONE draw, lane32(0x41, i, t) < T(p_infect) (Listing 2); an infected
 * agent recovers iff lane32(0x43, i, t) < T(p_recover); R stays R. */
void orc_sirs_step(int64_t n, const int32_t* row_ptr, const int32_t* col, uint64_t seed, uint32_t t,
                   uint64_t t_inf, uint64_t t_rec, const uint8_t* x, uint8_t* x_next)
{
    for (int64_t s = 0; s < n; ++s) {
        if (x[s] == ORC_S) {
            int exposed = 0;
            for (int32_t p = row_ptr[s]; p < row_ptr[s + 1]; ++p)
                if (x[col[p]] == ORC_I) { exposed = 1; break; }
            int inf = exposed && (uint64_t)orc_lane32(seed, ORC_TAG_SIRS_TX, (uint64_t)s, t) < t_inf;
            x_next[s] = inf ? ORC_I : ORC_S;
        } else if (x[s] == ORC_I) {
            x_next[s] = ((uint64_t)orc_lane32(seed, ORC_TAG_SIRS_REC, (uint64_t)s, t) < t_rec) ? ORC_R : ORC_I;
        } else {
            x_next[s] = ORC_R;
        }
    }
}

int orc_sirs_run(int64_t n, const int32_t* row_ptr, const int32_t* col, uint64_t seed, double p_inf,
                 double p_rec, uint32_t t0, int64_t steps, uint8_t* state, int64_t* counts_out)
{
    uint8_t* tmp = (uint8_t*)malloc((size_t)(n > 0 ? n : 1));
    if (!tmp) return ORC_E_OOM;
    uint64_t ti = orc_bernoulli_threshold(p_inf), tr = orc_bernoulli_threshold(p_rec);
    for (int64_t k = 0; k < steps; ++k) {
        orc_sirs_step(n, row_ptr, col, seed, t0 + (uint32_t)k, ti, tr, state, tmp);
        memcpy(state, tmp, (size_t)n);
        if (counts_out) {
            int64_t cc[3] = {0, 0, 0};
            for (int64_t i = 0; i < n; ++i) cc[state[i]] += 1;
            counts_out[3 * k] = cc[0];
            counts_out[3 * k + 1] = cc[1];
            counts_out[3 * k + 2] = cc[2];
        }
    }
    free(tmp);
    return 0;
}
