// SPDX-License-Identifier: Apache-2.0
//
// etaplab_b200.hpp — header-only C++ adapter that puts the B200 ETAP MLA decode path behind
// the reference's own entry point
//
//   etaplab::AttentionOutput etaplab::run_etap(const AttentionProblem&, const TileConfig&,
//                                              const BlockHook& = {}, const EtapFaults& = {});
//   (/root/reference/proj/include/etaplab/etap.hpp:47-48, src/etap.cpp:102-148)
//
// It is a template over the problem / output / tile types so it compiles against the
// reference's headers (etaplab::AttentionProblem, AttentionOutput, TileConfig, EtapFaults)
// without this repository depending on them. The only link dependency is libetap_mla.so
// (include/etap_mla.h).
//
// Semantics (mirroring the reference's error behaviour):
//   * tile fields < 1            -> std::invalid_argument (etap.cpp:104-106)
//   * d_qk != 576, d_v != 512, or V not equal to K[:, :512] (MLA latent aliasing)
//                                -> std::invalid_argument (outside the GPU path's scope)
//   * precision != exact64       -> std::invalid_argument: the GPU computes bf16 x bf16 -> fp32
//                                   on the stored operands, a mapping of exact64 storage only;
//                                   fp32 / fp16emu (matrix.hpp:22) are not emulated
//   * CUDA failure / no B200     -> std::runtime_error (there is no CPU fallback)
//   * BlockHook                  -> the device cannot call back per KV block: it records its
//                                   softmax state (one split, the reference's serial block
//                                   order, eager rescale) and the hook is replayed after the run
//                                   exactly as run_etap calls it (etap.cpp:115-129): query blocks
//                                   of b_r rows outer, KV blocks of b_c rows inner, BlockStepInfo
//                                   {query_block, kv_block, m_old, SoftmaxState{m, l}, rescale}
//                                   over the block's r rows (tiled_standard.hpp:32-40), for any
//                                   b_r / b_c (etap_mla_run_etap_f64_state)
//   * EtapFaults::negate_rescale -> ETAP_FLAG_NEGATE_RESCALE (same fault, on the device)
// Q/K are rounded to bf16 (RNE) on the way in, O and L are widened from fp32 on the way out;
// the reference's oracle (attention_ref) evaluated on the same rounded operands is the
// parity target (RMSE <= 2e-5).
#pragma once

#include <algorithm>
#include <cstddef>
#include <functional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "etap_mla.h"

namespace etaplab_b200 {

// Generic form: Output must be default-constructible with members `o` (a Matrix-like type
// constructible from (rows, cols) with data()) and `l` (a std::vector<double>-like type).
template <class Problem>
int precision_of(const Problem& p) {
    return static_cast<int>(p.precision);  // etaplab::Precision {exact64, fp32, fp16emu}
}

[[noreturn]] inline void raise(int rc) {
    if (rc == ETAP_ERR_SHAPE) throw std::invalid_argument(etap_mla_last_error());
    throw std::runtime_error(std::string("etap_b200: ") + etap_mla_last_error());
}

template <class Output, class Problem, class Tiles, class Faults>
Output run_etap(const Problem& p, const Tiles& tiles, const Faults& faults) {
    using MatrixT = decltype(Output{}.o);
    Output out;
    out.o = MatrixT(p.n_q, p.d_v);
    out.l.assign(p.n_q, 0.0);
    const unsigned flags = faults.negate_rescale ? ETAP_FLAG_NEGATE_RESCALE : 0u;
    const int rc = etap_mla_run_etap_f64(
        p.q.data(), static_cast<int64_t>(p.n_q), p.k.data(), static_cast<int64_t>(p.n_kv),
        static_cast<int64_t>(p.d_qk), p.v.data(), static_cast<int64_t>(p.d_v), p.scale, precision_of(p),
        static_cast<int64_t>(tiles.b_r), static_cast<int64_t>(tiles.b_c),
        static_cast<int64_t>(tiles.stages), flags, out.o.data(), out.l.data());
    if (rc != ETAP_OK) raise(rc);
    return out;
}

namespace detail {
// BlockStepInfo from the hook's signature (etaplab::BlockHook = std::function<void(const BlockStepInfo&)>)
template <class F>
struct hook_arg;
template <class R, class A>
struct hook_arg<std::function<R(A)>> {
    using type = std::remove_cv_t<std::remove_reference_t<A>>;
};
}  // namespace detail

// Reference-signature form: drop-in for etaplab::run_etap(problem, tiles, hook, faults).
template <class Output, class Problem, class Tiles, class Hook, class Faults>
Output run_etap(const Problem& p, const Tiles& tiles, const Hook& hook, const Faults& faults) {
    if (!hook) return run_etap<Output>(p, tiles, faults);
    using Info = typename detail::hook_arg<Hook>::type;
    using State = std::remove_cv_t<std::remove_reference_t<decltype(std::declval<const Info&>().state)>>;
    if (tiles.b_r < 1 || tiles.b_c < 1 || tiles.stages < 1)
        throw std::invalid_argument("tile config fields must be >= 1");
    using MatrixT = decltype(Output{}.o);
    Output out;
    out.o = MatrixT(p.n_q, p.d_v);
    out.l.assign(p.n_q, 0.0);
    const std::size_t t_c = (p.n_kv + tiles.b_c - 1) / tiles.b_c;
    std::vector<double> state(t_c * 4 * p.n_q);
    // the reference's per-block rescale order (etap.cpp:40-47) so every step's factor is observable
    const unsigned flags = ETAP_FLAG_EAGER_RESCALE | (faults.negate_rescale ? ETAP_FLAG_NEGATE_RESCALE : 0u);
    const int rc = etap_mla_run_etap_f64_state(
        p.q.data(), static_cast<int64_t>(p.n_q), p.k.data(), static_cast<int64_t>(p.n_kv),
        static_cast<int64_t>(p.d_qk), p.v.data(), static_cast<int64_t>(p.d_v), p.scale, precision_of(p),
        static_cast<int64_t>(tiles.b_c), flags, out.o.data(), out.l.data(), state.data());
    if (rc != ETAP_OK) raise(rc);
    // state[j][0..3][row]: m_old, m, rescale, l after KV block j (include/etap_mla.h); replayed
    // in run_etap's order: query blocks of b_r rows outer, KV blocks inner (etap.cpp:115-129)
    for (std::size_t i0 = 0, qb = 0; i0 < p.n_q; i0 += tiles.b_r, ++qb) {
        const std::size_t i1 = std::min<std::size_t>(p.n_q, i0 + tiles.b_r);
        for (std::size_t j = 0; j < t_c; ++j) {
            auto row = [&](int r) {
                const double* b = state.data() + (j * 4 + r) * p.n_q;
                return std::vector<double>(b + i0, b + i1);
            };
            const std::vector<double> m_old = row(0), rescale = row(2);
            const State st{row(1), row(3)};
            hook(Info{qb, j, m_old, st, rescale});
        }
    }
    return out;
}

}  // namespace etaplab_b200
