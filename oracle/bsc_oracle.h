/* TEST INFRASTRUCTURE ONLY — the parity oracle, never the product.
 *
 * Plain-C restatement of the reference BSC truncated-EM path
 * (/root/reference/proj/src/linear_discrete.cpp:202-427, truncation.cpp:38-169,
 * core.cpp:36-76, parallel.cpp:27-158, model.cpp:187-220, bars.cpp:33-65),
 * evaluated in the same summation orders as the reference compiled against
 * oracle/eigen_shim (see that header). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / reference leg may load it.
 *
 * Status codes follow prsp_status (prsp.h:39-45): 0 ok, 2 config, 3 data,
 * 4 numeric, 5 internal; the message is in bsc_last_error() (per thread).
 */
#ifndef BSC_ORACLE_H
#define BSC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* bsc_last_error(void);

/* RngStream (core.hpp:129-150): mt19937_64 + 53-bit uniforms + Box-Muller. */
int bsc_rng_normals(uint64_t base_seed, uint64_t index, int derived, uint64_t n,
                    double* out);
int bsc_rng_uniforms(uint64_t seed, uint64_t n, double* out);

/* Data fixtures. */
int bsc_make_bars(uint32_t size, uint64_t n, double prob, double amplitude,
                  double noise, int max_mode, uint64_t seed, double* y_out,
                  double* truth_out);
int bsc_generate(uint32_t d, uint32_t h, const double* w, double pi,
                 double sigma2, uint64_t n, uint64_t seed, double* y_out);
int bsc_random_dictionary(uint32_t d, uint32_t h, uint64_t seed, double scale,
                          double* w_out);
int bsc_baseline_init(uint32_t d, uint32_t h, const double* y, uint64_t n,
                      uint64_t seed, double* w_out, double* pi_out,
                      double* sigma2_out);
int bsc_standard_init(uint32_t d, uint32_t h, uint32_t hprime, const double* y,
                      uint64_t n, uint64_t seed, double* w_out, double* pi_out,
                      double* sigma2_out);
int bsc_data_mean_variance(const double* y, uint64_t n, uint32_t d, double* out);

/* Truncation engine. */
int bsc_select_candidates(const double* scores, uint32_t h, uint32_t hprime,
                          uint32_t* out);
int bsc_state_count(uint32_t h, uint32_t hprime, uint32_t gamma, uint64_t* out);
int bsc_enumerate_binary(const uint32_t* cand, uint32_t hprime, uint32_t h,
                         uint32_t gamma, double* out, uint64_t* count);
int bsc_log_sum_exp(const double* v, uint64_t n, double* out);

/* Model. scalars[3] = {sum_y2, log_partition, points}. */
int bsc_log_joint(uint32_t d, uint32_t h, const double* w, double pi,
                  double sigma2, const double* y, const double* s, double* out);
int bsc_estep_stats(uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                    const double* w, double pi, double sigma2,
                    double temperature, const double* y, uint64_t n,
                    uint64_t row_begin, uint64_t row_end, double* sum_s,
                    double* sum_ssT, double* sum_y_sT, double* value_counts,
                    double* scalars);
int bsc_mstep(uint32_t d, uint32_t h, const double* w_prev, double pi_prev,
              double sigma2_prev, const double* sum_s, const double* sum_ssT,
              const double* sum_y_sT, const double* value_counts,
              const double* scalars, double* w_out, double* pi_out,
              double* sigma2_out);
int bsc_step(uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
             const double* w, double pi, double sigma2, double temperature,
             const double* y, uint64_t n, uint32_t shards, uint32_t workers,
             double* w_out, double* pi_out, double* sigma2_out,
             double* free_energy);
int bsc_candidates(uint32_t d, uint32_t h, uint32_t hprime, const double* w,
                   double pi, double sigma2, const double* y, uint64_t n,
                   uint32_t* out);
int bsc_inference(uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                  const double* w, double pi, double sigma2, const double* y,
                  uint64_t n, double* map_states, double* map_mass,
                  double* expected);
int bsc_exact_log_likelihood(uint32_t d, uint32_t h, const double* w, double pi,
                             double sigma2, const double* y, uint64_t n,
                             double* out);

/* Linear discrete families (linear_discrete.cpp): family 0 = bsc, 1 = tsc,
 * 2 = dsc. `alpha`/`probs`/`nalpha`: the dsc alphabet (ascending, contains 0)
 * and its probabilities (NULL/0 otherwise); `pi` for bsc/tsc. value_counts
 * has one entry per non-zero value; probs_out (dsc) is aligned with alpha. */
int ld_state_count(uint32_t h, uint32_t hprime, uint32_t gamma, uint32_t nv, uint64_t* out);
int ld_estep_stats(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
                   double pi, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                   const double* w, double sigma2, double temperature, const double* y,
                   uint64_t n, uint64_t row_begin, uint64_t row_end, double* sum_s,
                   double* sum_ssT, double* sum_y_sT, double* value_counts, double* scalars);
int ld_mstep(uint32_t family, const double* alpha, uint32_t nalpha, uint32_t d, uint32_t h,
             const double* w_prev, const double* sum_s, const double* sum_ssT,
             const double* sum_y_sT, const double* value_counts, const double* scalars,
             double* w_out, double* pi_out, double* probs_out, double* sigma2_out);
int ld_step(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
            double pi, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
            const double* w, double sigma2, double temperature, const double* y, uint64_t n,
            uint32_t shards, uint32_t workers, double* w_out, double* pi_out,
            double* probs_out, double* sigma2_out, double* free_energy);
int ld_candidates(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
                  double pi, uint32_t d, uint32_t h, uint32_t hprime, const double* w,
                  double sigma2, const double* y, uint64_t n, uint32_t* out);
int ld_inference(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
                 double pi, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                 const double* w, double sigma2, const double* y, uint64_t n,
                 double* map_states, double* map_mass, double* expected);
int ld_exact_log_likelihood(uint32_t family, const double* alpha, const double* probs,
                            uint32_t nalpha, double pi, uint32_t d, uint32_t h,
                            const double* w, double sigma2, const double* y, uint64_t n,
                            double* out);
int ld_generate(uint32_t family, const double* alpha, const double* probs, uint32_t nalpha,
                double pi, uint32_t d, uint32_t h, const double* w, double sigma2, uint64_t n,
                uint64_t seed, double* y_out);

/* Max causes (max_causes.cpp): mode 0 = mca (max), 1 = mmca (absmax); rho =
 * soft winner exponent (mca only). estep scalars = {sum_act, log_partition,
 * points}; winner_num / winner_den are D×H. */
int mca_estep_stats(uint32_t mode, double rho, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                    const double* w, double pi, double sigma2, double temperature, const double* y, uint64_t n,
                    uint64_t row_begin, uint64_t row_end, double* winner_num, double* winner_den,
                    double* scalars);
int mca_mstep_fixedpoint(uint32_t mode, uint32_t d, uint32_t h, const double* w_prev, const double* winner_num,
                         const double* winner_den, const double* scalars, double* w_out, double* pi_out);
int mca_step(uint32_t mode, double rho, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
             const double* w, double pi, double sigma2, double temperature, const double* y, uint64_t n,
             uint32_t shards, uint32_t workers, double* w_out, double* pi_out, double* sigma2_out,
             double* free_energy);
int mca_candidates(uint32_t mode, uint32_t d, uint32_t h, uint32_t hprime, const double* w, double pi,
                   double sigma2, const double* y, uint64_t n, uint32_t* out);
int mca_inference(uint32_t mode, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma, const double* w,
                  double pi, double sigma2, const double* y, uint64_t n, double* map_states, double* map_mass,
                  double* expected);
int mca_log_joint(uint32_t mode, uint32_t d, uint32_t h, const double* w, double pi, double sigma2,
                  const double* y, const double* s, double* out);
int mca_exact_log_likelihood(uint32_t mode, uint32_t d, uint32_t h, const double* w, double pi, double sigma2,
                             const double* y, uint64_t n, double* out);
int mca_generate(uint32_t mode, uint32_t d, uint32_t h, const double* w, double pi, double sigma2, uint64_t n,
                 uint64_t seed, double* y_out);
int mca_standard_init(uint32_t mode, uint32_t d, uint32_t h, uint32_t hprime, const double* y, uint64_t n,
                      uint64_t seed, double* w_out, double* pi_out, double* sigma2_out);

#ifdef __cplusplus
}
#endif

#endif /* BSC_ORACLE_H */
