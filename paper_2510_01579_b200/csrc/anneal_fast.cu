// Dispatch of the throughput CIM-CAC anneal (kernel and its description in
// anneal_fast_impl.cuh; one instantiation unit per register layout).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "anneal_fast_impl.cuh"

namespace il {

using namespace fastk;

namespace {
// Register layouts built: N = 8 NT spins per half for these NT; a problem of
// n spins runs on the smallest N >= n (inert padding spins, see k_anneal_fast).
constexpr int kFastNT[] = {1, 2, 3, 4, 5, 6, 7, 8};
int fast_nt_for(int n) {
    for (int nt : kFastNT)
        if (8 * nt >= n) return nt;
    return 0;
}

}  // namespace

#ifndef IL_UMMA  // coupling product on tcgen05 (anneal_umma.cu) by default
#define IL_UMMA 0
#endif
// ISINGLINK_UMMA=0/1 overrides the build default (A/B measurements)
static bool use_umma() {
    static const int v = [] {
        const char* e = getenv("ISINGLINK_UMMA");
        return e && *e ? (atoi(e) != 0 ? 1 : 0) : IL_UMMA;
    }();
    return v != 0;
}

// Steps whose refreshes keep the third split pass (lo(v) x hi(G)): all of
// them in IL_PREC_FP32, the first kMixedFullSteps in IL_PREC_MIXED.  The
// dynamics are chaotic early on (rounding there changes trajectories) and
// contracting late: measured on 16,384 REs per configuration, dropping the
// pass from step 16 on keeps 99.95-99.99% of the decisions identical to
// FP64-exact (99.88-99.96% when dropped throughout).
// ISINGLINK_FULL_STEPS=k overrides for A/B runs.
constexpr int kMixedFullSteps = 16;
static int full_steps_for(int n_steps, int precision) {
    static const int v = [] {
        const char* e = getenv("ISINGLINK_FULL_STEPS");
        return e && *e ? atoi(e) : -1;
    }();
    if (v >= 0) return v;
    return precision == IL_PREC_MIXED ? std::min(kMixedFullSteps, n_steps) : n_steps;
}

bool fast_anneal_uses_umma(int N, int B) { return use_umma() && umma_anneal_supported(N, B); }

int fast_anneal_layout(int N) { return 8 * fast_nt_for(N); }

bool fast_anneal_supported(int N, int B, const AnnealScalars& s) {
    if (N < 1 || fast_nt_for(N) == 0 || B <= 0 || (B % 16 != 0 && B != 8)) return false;
    // the aux/initial-state check folds x0 into the sticky max: require |x0| < thr
    if (!(s.x0_range * 0.5 < s.thr)) return false;
    // e may not overflow FP32 while x stays below the threshold
    const double thr2 = s.thr * s.thr;
    const double r1 = fabs(1.0 + s.dt * s.zeta * s.a);
    const double r2 = fabs(1.0 - s.dt * s.zeta * (thr2 - s.a));
    const double rmax = fmax(r1, r2);
    if (rmax > 1.0 && (double)s.n_steps * log(rmax) > 80.0) return false;
    return true;
}

int launch_anneal_fast(const double* G, const double* g, const double* b,
                       const uint64_t* base_seed, const double* eps_p, int64_t P, int N, int B,
                       const AnnealScalars& s, int precision, int8_t* spins, uint8_t* diverged,
                       double* energies, cudaStream_t st, int screen_rows, int64_t* steps,
                       int64_t* mvms, int count_rows, const double* gstats) {
    if (!fast_anneal_supported(N, B, s)) {
        set_error("fast anneal kernel does not support n_dim=%d n_anneals=%d with these params", N, B);
        return IL_ERR_UNSUPPORTED;
    }
    if (P == 0) return IL_OK;
    FastScalars fs;
    fs.alpha = (float)(1.0 + s.dt * (s.p - 1.0));
    fs.ndt = (float)(-s.dt);
    fs.beta = (float)(1.0 + s.dt * s.zeta * s.a);
    fs.ndtz = (float)(-s.dt * s.zeta);
    fs.e_floor = (float)s.e_floor;
    fs.thr2 = (float)(s.thr * s.thr);
    fs.dt = s.dt;
    fs.x0_lo = s.x0_lo;
    fs.x0_range = s.x0_range;
    fs.f_mvm = s.f_mvm;
    fs.n_steps = s.n_steps;
    fs.sdt = sqrt(s.dt);
    fs.qthr = (float)(1.0 + s.dt * (s.p - 1.0) - s.dt * s.thr * s.thr);
    fs.b_valid = screen_rows;
    fs.b_out = count_rows;
    fs.full_steps = full_steps_for(s.n_steps, precision);
    fs.n_probs = P;
    fs.gstats = gstats;
    fs.rng = s.rng;
    fs.x0_lo_f = (float)s.x0_lo;
    fs.x0_range_f = (float)s.x0_range;
    IL_REQUIRE((steps == nullptr) == (mvms == nullptr) && (!steps || (count_rows > 0 && count_rows <= B)),
               "fast anneal: steps and mvms go together, for 1..B rows");
    // the screen pays off from N = 24 on (at N = 16 the FP64 epilogue is cheaper)
    // ISINGLINK_SCREEN=0 turns the screen off (the parity test compares both)
    static const bool screen_on = [] {
        const char* e = getenv("ISINGLINK_SCREEN");
        return !(e && *e == '0');
    }();
    const bool screened = screen_on && screen_rows > 0 && N >= 24;
    // lane part 1 of an anneal's two x0 lanes starts (2N + 2) / 2 draws into the stream
    pcg_jump((2 * N + 2) / 2, &fs.jump_mult[3], &fs.jump_add[3]);
    const bool split = precision != IL_PREC_TF32;
    // x and e share their per-step factor exactly when zeta*dt == dt and
    // 1 + dt (p - 1) == 1 + dt zeta a in FP32 (the reference defaults)
    // The scaled state (SAME_QR instantiations, IL_SCALED_X) tests divergence
    // on q = alpha - dt x^2 against alpha - dt thr^2: keep the test's
    // resolution (one ulp of q) below 2^-18 of dt thr^2, otherwise (tiny
    // thresholds) take the general instantiation, which compares x^2 directly.
    const bool same_qr = fs.alpha == fs.beta && fs.ndt == fs.ndtz &&
                         (!IL_SCALED_X || s.dt * s.thr * s.thr >= fabs((double)fs.alpha) * 0x1p-6);
    if (use_umma() && steps == nullptr && umma_anneal_supported(N, B))
        return launch_anneal_umma(G, g, b, base_seed, eps_p, P, N, B, &fs, split, same_qr, spins,
                                  diverged, energies, screened, st);
#define IL_NT(k) \
    case k: return launch_fast_nt##k(G, g, b, base_seed, eps_p, P, B, fs, split, same_qr, spins, diverged, energies, screened, N, steps, mvms, st)
    switch (fast_nt_for(N)) {
        IL_NT(1);
        IL_NT(2);
        IL_NT(3);
        IL_NT(4);
        IL_NT(5);
        IL_NT(6);
        IL_NT(7);
        IL_NT(8);
#undef IL_NT
        default:
            set_error("fast anneal kernel not instantiated for n_dim=%d", N);
            return IL_ERR_UNSUPPORTED;
    }
}

}  // namespace il
