/*
 * ORACLE — test infrastructure only.  Never linked into the product path.
 *
 * Plain-C restatement of the reference integration kernel
 *   reference: pkg/src/isinglink/_kernel.pyx:16-102 (run_anneals)
 *   contract:  pkg/src/isinglink/_kernel_py.py:24-92
 *
 * Explicit-Euler CIM-CAC dynamics for a batch of anneals over one shared
 * structured Ising problem (G, g_diag, b).  The arithmetic is written in the
 * exact evaluation order of the Cython-generated C for _kernel.pyx (checked
 * against `cython -3` output: _kernel.pyx:65-100), and this file must be
 * compiled with -ffp-contract=off so no multiply-add is fused.  Under those
 * rules its outputs are bit-identical to the reference "ext" backend, which
 * the CPU test-suite verifies against the compiled reference in oracle/_ref
 * and against the committed golden fixtures.
 *
 * Memory layout (all C-contiguous, row-major):
 *   G[n*n] f64, g_diag[n] f64, b[n] f64, x0[n_batch*(2n+1)] f64
 *   spins[n_batch*(2n+1)] i8, diverged[n_batch] u8, steps[n_batch] i64,
 *   mvms[n_batch] i64
 * Scratch (caller-owned, 4*(2n+1) doubles) keeps the oracle allocation-free.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

int cac_oracle_run_anneals(const double *G, const double *g_diag, const double *b,
                           const double *x0, int64_t n, int64_t n_batch,
                           double dt, double p, double a, double zeta, double eps,
                           double e_floor, int64_t f_mvm, int64_t n_steps,
                           double diverge_threshold, int8_t *spins,
                           uint8_t *diverged, int64_t *steps, int64_t *mvms,
                           double *scratch)
{
    const int64_t S = 2 * n + 1;
    double *x = scratch, *e = scratch + S, *cpl = scratch + 2 * S, *v = scratch + 3 * S;
    if (f_mvm < 1 || n < 0 || n_batch < 0) return -1;

    for (int64_t r = 0; r < n_batch; ++r) {
        diverged[r] = 0;
        steps[r] = n_steps;
        mvms[r] = 0;
        for (int64_t i = 0; i < S; ++i) {
            x[i] = x0[r * S + i];
            e[i] = 1.0;
            cpl[i] = 0.0;
        }
        for (int64_t t = 0; t < n_steps; ++t) {
            if (t % f_mvm == 0) {
                /* refresh: v = x1 + x2, cpl = [G v - g.x1 + b xa; G v - g.x2 + b xa; b.v] */
                double xa = x[2 * n];
                double bdot = 0.0;
                for (int64_t i = 0; i < n; ++i) {
                    v[i] = x[i] + x[n + i];
                    bdot = bdot + b[i] * v[i];
                }
                for (int64_t i = 0; i < n; ++i) {
                    double acc = 0.0;
                    for (int64_t j = 0; j < n; ++j) acc = acc + G[i * n + j] * v[j];
                    cpl[i] = (acc - g_diag[i] * x[i]) + b[i] * xa;
                    cpl[n + i] = (acc - g_diag[i] * x[n + i]) + b[i] * xa;
                }
                cpl[2 * n] = bdot;
                mvms[r] += 1;
            }
            int bad = 0;
            for (int64_t i = 0; i < S; ++i) {
                double xi = x[i], ei = e[i];
                double dxi = (((p - 1.0) * xi) - ((xi * xi) * xi)) - ((eps * ei) * cpl[i]);
                double dei = ((-zeta) * ((xi * xi) - a)) * ei;
                xi = xi + dt * dxi;
                ei = ei + dt * dei;
                if (ei < e_floor) ei = e_floor;
                x[i] = xi;
                e[i] = ei;
                if (fabs(xi) > diverge_threshold || !isfinite(xi) || !isfinite(ei)) bad = 1;
            }
            if (bad) {
                diverged[r] = 1;
                steps[r] = t + 1;
                break;
            }
        }
        for (int64_t i = 0; i < S; ++i) spins[r * S + i] = (x[i] >= 0.0) ? 1 : -1;
    }
    return 0;
}
