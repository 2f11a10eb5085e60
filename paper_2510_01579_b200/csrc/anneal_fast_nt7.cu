// k_anneal_fast instantiations for the register layout NT = 7 (N = 56 spins per half).
#include "anneal_fast_impl.cuh"

namespace il {
IL_FAST_NT_DECL(7) {
    return fast_impl::launch_nt<7>(G, g, b, base_seed, eps_p, P, B, fs, split, same_qr, spins, diverged,
                                    energies, screened, n_rt, steps, mvms, st);
}
}  // namespace il
