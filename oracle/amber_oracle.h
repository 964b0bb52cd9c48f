/*
 * amber_oracle.h -- TEST INFRASTRUCTURE ONLY (see amber_oracle.c).
 * Private to oracle/: nothing in paper_2601_16292_b200/ includes this file.
 */
#ifndef AMBER_ORACLE_H
#define AMBER_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* R5: stream tags (counter word 3). */
enum {
    ORC_TAG_WEALTH_RECV = 0x01,
    ORC_TAG_SIR_TX = 0x10,
    ORC_TAG_SIR_REC = 0x11,
    ORC_TAG_SIR_INIT = 0x12,
    ORC_TAG_GRAPH = 0x13,
    ORC_TAG_BOIDS_POS = 0x20,
    ORC_TAG_BOIDS_VEL = 0x21,
    ORC_TAG_WALK_POS = 0x30,
    ORC_TAG_WALK_VEL = 0x31,
    ORC_TAG_SIRS_POS = 0x40,
    ORC_TAG_SIRS_TX = 0x41,
    ORC_TAG_SIRS_INIT = 0x42,
    ORC_TAG_SIRS_REC = 0x43
};

enum { ORC_S = 0, ORC_I = 1, ORC_R = 2 };
enum { ORC_E_INVALID = -1, ORC_E_OOM = -2 };

typedef struct {
    float L, R, rs, wc, wa, ws, vmax, dt;
} orc_boids_params;

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t orc_lane64(uint64_t seed, uint32_t tag, uint64_t u, uint32_t t);
uint32_t orc_lane32(uint64_t seed, uint32_t tag, uint64_t u, uint32_t t);
uint64_t orc_mulhi64(uint64_t x, uint64_t n);
uint64_t orc_bernoulli_threshold(double p);
float orc_u01(uint32_t x);
int64_t orc_round_count(double x);
uint64_t orc_mix64(uint64_t z);
uint64_t orc_digest_bits32(const uint32_t* bits, int64_t n, int64_t id0);
uint64_t orc_digest_u8(const uint8_t* v, int64_t n, int64_t id0);

int64_t orc_wealth_receiver(uint64_t seed, int64_t n, int64_t i, uint32_t t, int exclude_self);
int orc_wealth_step(int64_t n, int32_t amount, int exclude_self, uint64_t seed, uint32_t t,
                    const int32_t* w, int32_t* w_next);
int orc_wealth_run(int64_t n, int32_t amount, int exclude_self, uint64_t seed, uint32_t t0,
                   int64_t steps, int32_t* w, int64_t* total_out, int64_t* active_out,
                   uint64_t* digest_out);

void orc_er_draw(uint64_t seed, int64_t n, int64_t e, int64_t* u_out, int64_t* v_out);
int64_t orc_er_graph(int64_t n, int64_t m, uint64_t seed, int32_t* row_ptr, int32_t* col);

int orc_sir_init(int64_t n, int64_t k, uint64_t seed, uint8_t* state);
uint32_t orc_sir_tx_word(uint64_t seed, int64_t a, int64_t b, uint32_t t);
void orc_sir_step(int64_t n, const int32_t* row_ptr, const int32_t* col, uint64_t seed,
                  uint32_t t, uint64_t t_beta, uint64_t t_gamma, const uint8_t* x,
                  uint8_t* x_next);
int orc_sir_run(int64_t n, const int32_t* row_ptr, const int32_t* col, uint64_t seed,
                double beta, double gamma, uint32_t t0, int64_t steps, uint8_t* state,
                int64_t* counts_out, uint64_t* digest_out);
int64_t orc_sir_replicate(int64_t n, double mean_degree, double beta, double gamma,
                          double init_frac, uint64_t seed, int64_t steps);
int orc_sir_sweep(int64_t n, double mean_degree, double gamma, double init_frac,
                  int64_t n_reps, const double* betas, const uint64_t* seeds, int64_t steps,
                  double* out_final_r_frac);

void orc_boids_init(int64_t n, float L, uint64_t seed, float* px, float* py, float* vx, float* vy);
void orc_boids_step_brute(int64_t n, const orc_boids_params* P, const float* px, const float* py,
                          const float* vx, const float* vy, float* opx, float* opy, float* ovx,
                          float* ovy);
void orc_boids_step_brute_sample(int64_t n, const orc_boids_params* P, const float* px,
                                 const float* py, const float* vx, const float* vy,
                                 int64_t n_sample, const int64_t* ids, float* opx, float* opy,
                                 float* ovx, float* ovy, int64_t* n_neigh);
int orc_boids_step_binned(int64_t n, const orc_boids_params* P, const float* px, const float* py,
                          const float* vx, const float* vy, float* opx, float* opy, float* ovx,
                          float* ovy);
void orc_boids_metrics(int64_t n, const float* vx, const float* vy, double* mean_speed,
                       double* polarisation);
int orc_boids_run(int64_t n, const orc_boids_params* P, int64_t steps, float* px, float* py,
                  float* vx, float* vy, double* mean_speed_out, double* polar_out);
void orc_boids_step_brute_f64(int64_t n, const orc_boids_params* P, const double* px,
                              const double* py, const double* vx, const double* vy, double* opx,
                              double* opy, double* ovx, double* ovy);

void orc_walk_init(int64_t n, float L, uint64_t seed, float* px, float* py);
void orc_walk_step(int64_t n, float L, float vmax, uint64_t seed, uint32_t t, const float* px, const float* py,
                   float* opx, float* opy);
int orc_walk_run(int64_t n, float L, float vmax, uint64_t seed, uint32_t t0, int64_t steps, float* px, float* py,
                 const float* ox, const float* oy, double* mean_disp_out);

int orc_sirs_init(int64_t n, float L, int64_t k, uint64_t seed, float* px, float* py, uint8_t* state);
int64_t orc_sirs_contacts(int64_t n, const float* px, const float* py, float r, int32_t* row_ptr, int32_t* col,
                          int64_t cap);
int64_t orc_sirs_contacts_grid(int64_t n, const float* px, const float* py, float L, float r, int32_t* row_ptr,
                               int32_t* col, int64_t cap);
void orc_sirs_step(int64_t n, const int32_t* row_ptr, const int32_t* col, uint64_t seed, uint32_t t,
                   uint64_t t_inf, uint64_t t_rec, const uint8_t* x, uint8_t* x_next);
int orc_sirs_run(int64_t n, const int32_t* row_ptr, const int32_t* col, uint64_t seed, double p_inf,
                 double p_rec, uint32_t t0, int64_t steps, uint8_t* state, int64_t* counts_out);

#ifdef __cplusplus
}
#endif
#endif
