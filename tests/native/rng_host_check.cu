// Host-side harness for csrc/rng_numpy.cuh (compiled by nvcc as host code,
// runs on CPU).  Reads "n_parts p0 p1 ..." lines or "x0 seed S" lines from
// stdin and prints derive_seed values / uniform(-0.1, 0.1) draws as hex bits.
#include <stdio.h>
#include <string.h>
#include <inttypes.h>
#include "../../paper_2510_01579_b200/csrc/rng_numpy.cuh"

int main() {
    char kind[16];
    while (scanf("%15s", kind) == 1) {
        if (!strcmp(kind, "seed")) {
            int n; uint64_t p[6];
            if (scanf("%d", &n) != 1) return 1;
            for (int i = 0; i < n; ++i) if (scanf("%" SCNu64, &p[i]) != 1) return 1;
            printf("%" PRIu64 "\n", il::derive_seed(p, n));
        } else if (!strcmp(kind, "x0")) {
            uint64_t s; int S;
            if (scanf("%" SCNu64 " %d", &s, &S) != 2) return 1;
            il::Pcg64 r; r.seed_from(s);
            for (int k = 0; k < S; ++k) {
                double v = r.uniform(-0.1, 0.1 - (-0.1));
                uint64_t bits; memcpy(&bits, &v, 8);
                printf("%016" PRIx64 "%c", bits, k + 1 == S ? '\n' : ' ');
            }
        } else if (!strcmp(kind, "jump")) {
            // check advance-by-k against k single steps
            uint64_t s; int k;
            if (scanf("%" SCNu64 " %d", &s, &k) != 2) return 1;
            il::Pcg64 a, b; a.seed_from(s); b.seed_from(s);
            const il::U128 M = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
            il::U128 pm = {0, 1}, sum = {0, 0};
            for (int i = 0; i < k; ++i) { sum = il::add128(sum, pm); pm = il::mul128(pm, M); }
            for (int i = 0; i < k; ++i) a.step();
            b.state = il::add128(il::mul128(b.state, pm), il::mul128(b.inc, sum));
            printf("%d\n", a.state.hi == b.state.hi && a.state.lo == b.state.lo);
        }
    }
    return 0;
}
