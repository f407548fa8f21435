// inst.cuh — one fused-kernel shape per translation unit (inst_*.cu): the
// kernel table entry (ghc_internal.cuh LstmEntry) of lstm(D,H,T)→softmax(H,K)
// or of an LSTM trunk, with every kernel variant instantiated here.
#pragma once

#include "ghc_internal.cuh"

namespace ghc_inst {

template <int D, int H, int T, int K, int CS, bool TC>
constexpr void (*tc_fn())(StepArgs) {
  if constexpr (TC) return &lstm_round_tc_kernel<D, H, T, K, CS>;
  else return nullptr;
}

// the per-worker-gradient variant (MULTI: session sync EASGD; head shapes, clusters of 4)
template <int D, int H, int T, int K, bool HEAD>
constexpr void (*multi_fn())(StepArgs) {
  if constexpr (HEAD) return &lstm_round_kernel<D, H, T, K, 4, false, true>;
  else return nullptr;
}

// the resident-service variant of the round kernel (head shapes only)
template <int D, int H, int T, int K, int CS, bool HEAD>
constexpr void (*res_fn())(StepArgs) {
  if constexpr (HEAD) return &lstm_round_kernel<D, H, T, K, CS, true>;
  else return nullptr;
}

template <int D, int H, int T, int K, bool TC = true>
LstmEntry make_entry(const char* name) {
  using N = LstmNet<D, H, T, K>;
  using R4 = RoundLayout<D, H, T, K, 4>;
  using R8 = RoundLayout<D, H, T, K, 8>;
  using R2 = RoundLayout<D, H, T, K, 2>;
  using C4 = TcLayout<D, H, T, K, 4>;
  using C8 = TcLayout<D, H, T, K, 8>;
  static_assert(C4::EP == R4::EP && C8::EP == R8::EP, "same partial-row layout");
  return LstmEntry{D,
                   H,
                   T,
                   K,
                   &lstm_softmax_step_kernel<D, H, T, K>,
                   {&lstm_round_kernel<D, H, T, K, 4>, &lstm_round_kernel<D, H, T, K, 8>,
                    &lstm_round_kernel<D, H, T, K, 2>},
                   {res_fn<D, H, T, K, 4, TC>(), res_fn<D, H, T, K, 8, TC>(), res_fn<D, H, T, K, 2, TC>()},
                   {tc_fn<D, H, T, K, 4, TC>(), tc_fn<D, H, T, K, 8, TC>(), nullptr},
                   {multi_fn<D, H, T, K, TC>(), nullptr, nullptr},
                   N::P,
                   N::PPAD,
                   {R4::EP, R8::EP, R2::EP},
                   &N::smem_bytes,
                   {&R4::smem_bytes, &R8::smem_bytes, &R2::smem_bytes},
                   {&C4::smem_bytes, &C8::smem_bytes, nullptr},
                   name};
}

}  // namespace ghc_inst

#define GHC_INST(D, H, T, K)                                              \
  LstmEntry ghc_entry_##D##_##H##_##T##_##K() {                           \
    return ghc_inst::make_entry<D, H, T, K>("lstm_round<D" #D ",H" #H ",T" #T ",K" #K ">"); \
  }
#define GHC_INST_TRUNK(D, H, T)                                                  \
  LstmEntry ghc_trunk_##D##_##H##_##T() {                                        \
    return ghc_inst::make_entry<D, H, T, 1, false>("lstm_trunk<D" #D ",H" #H ",T" #T ">"); \
  }
