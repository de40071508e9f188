/*
 * oracle/sv.c -- plain fp64 state-vector oracle for arXiv:2111.03011's sparse-state
 * sliced contraction.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header or table with the product (paper_2111_03011_b200/csrc); it reads the same
 * seeded circuit description (tn_inputs/) and nothing else.
 *
 * What it computes (SURVEY §8(c) "Definition"):
 *   psi = U_C |0^n>, where each gate of the circuit is applied in circuit order and,
 *   right after the k-th gate touching qubit q (k counts EVERY gate on q, single- and
 *   two-qubit, 1-based), every "insertion" registered on wire (q,k)
 *   is applied:
 *       op 0 : projector Pi_0 = |0><0| on qubit q  (slice value 0)
 *       op 1 : projector Pi_1 = |1><1| on qubit q  (slice value 1)
 *       op 2 : sigma_z on qubit q                 (E = I/2 + sigma_z/2)
 *   Contracting the network with sliced edge (q,k) fixed to v is exactly inserting Pi_v
 *   on that wire (sum over v of Pi_v = I, "The summation of all sub-tasks
 *   results will return the contraction output of the original tensor network").
 *
 * Conventions: qubit q is bit (n-1-q) of the state index (qubit 0 = MSB);
 * single-qubit matrices are U[out][in]; fSim acts on local index 2*x_a + x_b for targets
 * (a, b) with the matrix of PAPER.md Eq. (1), L96-L102.
 *
 * Plain loops only (one pass over the vector per gate, no fusion, no blocking); the
 * amplitude loop of each pass is an OpenMP parallel-for so that 30-qubit runs finish.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

/* PAPER.md Eq. (1):
 *   fSim(theta, phi) = [[1, 0, 0, 0],
 *                       [0, cos t, -i sin t, 0],
 *                       [0, -i sin t, cos t, 0],
 *                       [0, 0, 0, e^{-i phi}]]                                    */
static void fsim_matrix(double theta, double phi, cplx U[4][4]) {
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++) U[r][c] = 0.0;
    U[0][0] = 1.0;
    U[1][1] = cos(theta);
    U[1][2] = -I * sin(theta);
    U[2][1] = -I * sin(theta);
    U[2][2] = cos(theta);
    U[3][3] = cexp(-I * phi);
}

/* exported for the tests: the oracle's own Eq. (1) matrix, row-major, (re, im) pairs */
void sv_fsim_matrix(double theta, double phi, double* out32) {
    cplx U[4][4];
    fsim_matrix(theta, phi, U);
    for (int r = 0; r < 4; r++)
        for (int c = 0; c < 4; c++) {
            out32[2 * (4 * r + c)] = creal(U[r][c]);
            out32[2 * (4 * r + c) + 1] = cimag(U[r][c]);
        }
}

static void apply_1q(cplx* psi, int n, int q, cplx U[2][2]) {
    const int64_t N = (int64_t)1 << n;
    const int64_t m = (int64_t)1 << (n - 1 - q);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        if (i & m) continue;
        cplx a0 = psi[i], a1 = psi[i | m];
        psi[i] = U[0][0] * a0 + U[0][1] * a1;
        psi[i | m] = U[1][0] * a0 + U[1][1] * a1;
    }
}

static void apply_2q(cplx* psi, int n, int qa, int qb, cplx U[4][4]) {
    const int64_t N = (int64_t)1 << n;
    const int64_t ma = (int64_t)1 << (n - 1 - qa);
    const int64_t mb = (int64_t)1 << (n - 1 - qb);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        if ((i & ma) || (i & mb)) continue;
        int64_t idx[4] = {i, i | mb, i | ma, i | ma | mb}; /* local index 2*x_a + x_b */
        cplx v[4], w[4];
        for (int c = 0; c < 4; c++) v[c] = psi[idx[c]];
        for (int r = 0; r < 4; r++) {
            w[r] = 0.0;
            for (int c = 0; c < 4; c++) w[r] += U[r][c] * v[c];
        }
        for (int r = 0; r < 4; r++) psi[idx[r]] = w[r];
    }
}

static void apply_insertion(cplx* psi, int n, int q, int op) {
    const int64_t N = (int64_t)1 << n;
    const int64_t m = (int64_t)1 << (n - 1 - q);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        int bit = (i & m) ? 1 : 0;
        if (op == 0 || op == 1) {
            if (bit != op) psi[i] = 0.0;
        } else if (op == 2) {
            if (bit) psi[i] = -psi[i];
        }
    }
}

/* Run the circuit with insertions; psi (2^n complex, caller-allocated, interleaved re/im)
 * receives the final state.  kind[g]: 0 = single-qubit gate with matrix u[8g..8g+7]
 * (U00, U01, U10, U11 as re/im pairs, U[out][in]); 1 = fSim(theta[g], phi[g]) on
 * (q0[g], q1[g]).  Returns 0 on success, -1 on bad arguments. */
int sv_run(int n, int n_gates, const int* kind, const int* q0, const int* q1,
           const double* theta, const double* phi, const double* u,
           int n_ins, const int* ins_q, const int* ins_k, const int* ins_op,
           int n_threads, double* psi_out) {
    if (n < 1 || n > 34) return -1;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
    const int64_t N = (int64_t)1 << n;
    cplx* psi = (cplx*)psi_out;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) psi[i] = 0.0;
    psi[0] = 1.0; /* |0^n> */
    int* count = (int*)calloc((size_t)n, sizeof(int));
    for (int g = 0; g < n_gates; g++) {
        int touched[2], nt = 0;
        if (kind[g] == 0) {
            cplx U[2][2] = {{u[8 * g] + I * u[8 * g + 1], u[8 * g + 2] + I * u[8 * g + 3]},
                            {u[8 * g + 4] + I * u[8 * g + 5], u[8 * g + 6] + I * u[8 * g + 7]}};
            if (q0[g] < 0 || q0[g] >= n) { free(count); return -1; }
            apply_1q(psi, n, q0[g], U);
            touched[nt++] = q0[g];
        } else {
            cplx U[4][4];
            if (q0[g] < 0 || q0[g] >= n || q1[g] < 0 || q1[g] >= n || q0[g] == q1[g]) { free(count); return -1; }
            fsim_matrix(theta[g], phi[g], U);
            apply_2q(psi, n, q0[g], q1[g], U);
            touched[nt++] = q0[g];
            touched[nt++] = q1[g];
        }
        for (int t = 0; t < nt; t++) {
            int q = touched[t];
            count[q] += 1;
            for (int s = 0; s < n_ins; s++)
                if (ins_q[s] == q && ins_k[s] == count[q]) apply_insertion(psi, n, q, ins_op[s]);
        }
    }
    free(count);
    return 0;
}

/* Same as sv_run but only returns psi at the M given indices (avoids a 2^n copy
 * to Python at n = 30).  amps_out: M complex (re, im). */
int sv_run_amps(int n, int n_gates, const int* kind, const int* q0, const int* q1,
                const double* theta, const double* phi, const double* u,
                int n_ins, const int* ins_q, const int* ins_k, const int* ins_op,
                int n_threads, int64_t M, const uint64_t* idx, double* amps_out,
                double* norm2_out) {
    const int64_t N = (int64_t)1 << n;
    double* psi = (double*)malloc((size_t)N * 2 * sizeof(double));
    if (!psi) return -2;
    int rc = sv_run(n, n_gates, kind, q0, q1, theta, phi, u, n_ins, ins_q, ins_k, ins_op, n_threads, psi);
    if (rc == 0) {
        for (int64_t j = 0; j < M; j++) {
            if (idx[j] >= (uint64_t)N) { rc = -1; break; }
            amps_out[2 * j] = psi[2 * idx[j]];
            amps_out[2 * j + 1] = psi[2 * idx[j] + 1];
        }
        if (norm2_out) {
            double s = 0.0;
            for (int64_t i = 0; i < 2 * N; i++) s += psi[i] * psi[i];
            *norm2_out = s;
        }
    }
    free(psi);
    return rc;
}
