/*
 * ssqa_host.h -- C entry points for the host-side problem builders of
 * libssqa_b200.so (no GPU needed).  They let non-C++ callers (the Python
 * tests and bench.py) build exactly the IsingModel the reference builds, then
 * hand it to ssqa_problem_create (include/ssqa_cuda.h).
 */
#ifndef SSQA_HOST_H
#define SSQA_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* qubo_to_ising(build_gi_qubo(generate_gi(n_nodes, edge_prob, seed, permute,
 * c1, c2))) -- gi.cpp:102-184, model.cpp:139-161.  h has n_nodes^2 entries,
 * J (n_nodes^2)^2 (dense, mirrored). */
int ssqa_gi_ising(int n_nodes, double edge_prob, uint64_t seed, int permute, double c1,
                  double c2, double* h, double* J, double* offset);

/* The host half of the device GI generator (ssqa_problem_create_gi): the
 * graph pair of generate_gi as 0/1 adjacency bytes adj[2*n_nodes^2] (graph 1,
 * then graph 2, 0-based) and the penalty's biases h[n_nodes^2] and offset in
 * closed form -- equal to ssqa_gi_ising's for dyadic c1, c2. */
int ssqa_gi_compact(int n_nodes, double edge_prob, uint64_t seed, int permute, double c1,
                    double c2, uint8_t* adj, double* h, double* offset);

/* BASELINE configs C4/C5, drawn from CounterRng
 * stream 8 (couplings) and 9 (biases) -- ids 1..7 are taken (rng.hpp:20-28).
 *   kind 0: J_ij = below(i*n+j, 16) - 8 for i<j, h_i = below(i, 16) - 8;
 *   kind 1: J_ij = raw(i*n+j) >> 63 ? +1 : -1 for i<j, h = 0. */
int ssqa_dense_ising(int n, int kind, uint64_t seed, double* h, double* J, double* offset);

/* ising_energy (model.cpp:112-126) of one +-1 state. */
int ssqa_ising_energy(int n, const double* h, const double* J, double offset,
                      const int8_t* spins, double* out);

const char* ssqa_host_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
