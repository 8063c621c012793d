/* bitlamb_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * C restatement of the reference's compression-stage hot path (1-bit LAMB,
 * arXiv 2104.06069 as implemented in /root/reference/proj).  It is the parity
 * checker for the B200 kernels and is never linked into the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * One source, two builds (oracle/Makefile):
 *   liboracle_f64.so  real = double, reductions in the reference's order
 *                     (kernels.cpp:134-150 blocked_sum).  Pinned bit-exactly
 *                     against the reference library itself (oracle/_ref) and
 *                     against the reference's known-answer tests.
 *   liboracle_f32.so  real = float, reductions in the B200 kernels' canonical
 *                     "tile-tree" order.  The GPU path must match
 *                     this build bit-for-bit; it is compared with the f64 build
 *                     and the reference within the fp32 tolerances of the tests.
 *
 * The API mirrors oracle/ref_shim.cpp (same oc_* names and status codes) so the
 * Python harness drives the reference and both oracle builds identically.
 * Status codes follow include/bitlamb_b200.h (bl_status).
 */
#ifndef BITLAMB_ORACLE_H_
#define BITLAMB_ORACLE_H_

#include <stdint.h>

#ifdef OC_REAL_FLOAT
typedef float oc_real;
#else
typedef double oc_real;
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OC_OK = 0,
  OC_DIMENSION = 1,
  OC_STAGE_ORDER = 2,
  OC_CONFIG = 3,
  OC_INVALID_ARGUMENT = 4,
  OC_RUNTIME = 5,
  OC_LOGIC = 6,
};

const char* oc_last_error(void);
int oc_real_bytes(void);

/* SimCluster (comm_sim.hpp:72-148) */
int oc_cluster_new(int n, uint64_t dim, int kind, int baseline_bits, int verify,
                   void** out);
void oc_cluster_set_tolerance(void* c, double tol);
void oc_cluster_free(void* c);
uint64_t oc_cluster_padded(void* c);
uint64_t oc_cluster_chunk(void* c);
int oc_cluster_compressed_allreduce(void* c, const oc_real* inputs, double es,
                                    oc_real* out);
int oc_cluster_compressed_allreduce_n(void* c, const oc_real* inputs, int n_inputs,
                                      uint64_t len, double es, oc_real* out);
int oc_cluster_lossless_allreduce(void* c, const oc_real* inputs, oc_real* out);
void oc_cluster_worker_error(void* c, int i, oc_real* out);
void oc_cluster_server_error(void* c, int j, oc_real* out);
void oc_cluster_ledger(void* c, uint64_t* out);
void oc_cluster_stats(void* c, double* out);
uint64_t oc_cluster_compensation_checks(void* c);
int oc_cluster_packet(void* c, int worker, int server, uint8_t* bytes);
int oc_cluster_server_packet(void* c, int server, uint8_t* bytes);

/* Per-rank phases of the same collective (used by the world_size>1 protocol
 * tests: worker i compresses its padded stream's n chunks, server j reduces the
 * n packets of chunk j).  Packets are sign bytes (serialize() layout) followed
 * by the scale as a native oc_real; for the f32 build that IS the wire layout. */
int oc_worker_compress(const oc_real* stream, uint64_t dim, int n, oc_real* werr,
                       double es, uint8_t* packets);
int oc_server_reduce(const uint8_t* packets, uint64_t chunk, int n, oc_real* serr,
                     double es, uint8_t* out_packet);
void oc_decompress(const uint8_t* packet, uint64_t len, oc_real* out);

/* free functions */
int oc_compress_with_feedback(const oc_real* v, oc_real* delta, uint64_t d, int kind,
                              double es, uint8_t* bytes, double* scale,
                              oc_real* decompressed);
int oc_volume_reduction(double w, double bb, double cb, double* out);
double oc_canonical_sum(const oc_real* x, uint64_t len, int kind); /* 0 |x|, 1 x^2 */

/* Optimizer (optimizers.hpp:93-145) */
int oc_opt_new(int variant, const uint64_t* sizes, int L, const double* hp,
               uint64_t total, uint64_t warmup, int scaled_ef, void** out);
void oc_opt_free(void* o);
int oc_opt_step(void* o, void* c, const oc_real* grads, int n, uint64_t t, double lr,
                double* trace, int* compressed);
void oc_opt_get(void* o, int which, oc_real* out);
void oc_opt_set(void* o, int which, const oc_real* in);
void oc_opt_get_scalars(void* o, double* out);
void oc_opt_set_scalars(void* o, const double* in);
int oc_opt_frozen(void* o);

#ifdef __cplusplus
}
#endif

#endif /* BITLAMB_ORACLE_H_ */
