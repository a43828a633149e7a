/* or_rng.h -- the oracle's own restatement of the restated GA's random stream
 * (test infrastructure only; see or_rng.c). */
#ifndef OR_RNG_H
#define OR_RNG_H
#include <stdint.h>

enum { OR_PH_INIT_U = 1, OR_PH_INIT_N = 2, OR_PH_BREED_U = 3, OR_PH_BREED_N = 4 };

typedef struct {
    uint64_t seed, ligand;  /* Philox key (global_seed, ligand_index), vd/ga.py:74-77 */
} or_rng_key;

void or_philox(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
uint64_t or_rng_word(const or_rng_key *key, int phase, int64_t gen, int64_t idx, int64_t slot);
double or_rng_uniform(uint64_t w);
uint64_t or_rng_below(uint64_t w, uint64_t n);
double or_rng_ln(double x);
double or_rng_cos_2pi(double u);
double or_rng_normal(const or_rng_key *key, int phase, int64_t gen, int64_t idx, int64_t comp);

#endif
