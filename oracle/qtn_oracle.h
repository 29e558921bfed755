/* oracle/qtn_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's bucket-elimination contraction
 * (the hot path), used exclusively by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the CHECKER.  The product never links it.
 *
 * Parity is pinned (not assumed): tests/test_oracle.py checks every function
 * here against golden vectors produced by the unmodified reference
 * (oracle/gen_golden.py -> tests/golden/).
 *
 * Complex numbers are interleaved (re, im) doubles; tensors are MSB-first
 * row-major over binary variables (reference proj/include/qtnsim/tensor.hpp:13-15).
 */
#ifndef QTN_ORACLE_H
#define QTN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference's exception types
 * (proj/include/qtnsim/errors.hpp:8-36). */
enum { QO_OK = 0, QO_INVALID = 1, QO_RESOURCE = 2, QO_SCHEDULE = 3, QO_NUMERICAL = 4 };

const char* qo_last_error(void);

/* NaiveBackend::contract (proj/src/engine.cpp:68-108).
 * ranks[t], vars = concatenated var lists, data = concatenated tensors.
 * Writes result vars (ascending) and data; returns the result rank or -status. */
int qo_contract_bucket(int n_tensors, const int* ranks, const int* vars,
                       const double* data, int n_sum, const int* sum_vars,
                       int* out_vars, double* out_data, int64_t out_cap);

/* contract_network (proj/src/engine.cpp:246-304) with contract_bucket's cap
 * check (engine.cpp:160-169) and the naive backend.
 * Schedule format (shared with the product's qtng_edge_schedule and the
 * reference wrapper ref_edge_schedule): for each bucket
 *   n_sum, sum_vars[n_sum], n_tensors, { rank, vars[rank] } * n_tensors
 * and `data` holds every tensor's entries in the same order.
 * Outputs the scalar, one (bucket_seq, width) record per non-empty bucket and
 * the peak result bytes. Returns QO_* status. */
int qo_contract_network(int n_buckets, const int* ints, const double* data,
                        int max_result_width, double* scalar_re_im,
                        int* rec_seq, int* rec_width, int rec_cap, int* n_records,
                        uint64_t* peak_bytes);

/* State-vector oracle: <C> for the QAOA ansatz on an n-vertex graph
 * (proj/src/statevector.cpp:25-84).  n <= 26. */
int qo_statevector_energy(int n, int m, const int* edges, int p, const double* gammas,
                          const double* betas, double* energy);

#ifdef __cplusplus
}
#endif
#endif
