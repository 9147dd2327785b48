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
//   * CUDA failure / no B200     -> std::runtime_error (there is no CPU fallback)
//   * BlockHook                  -> not observable on the GPU; a non-empty hook throws
//   * EtapFaults::negate_rescale -> ETAP_FLAG_NEGATE_RESCALE (same fault, on the device)
// Q/K are rounded to bf16 (RNE) on the way in, O and L are widened from fp32 on the way out;
// the reference's oracle (attention_ref) evaluated on the same rounded operands is the
// parity target (RMSE <= 2e-5).
#pragma once

#include <stdexcept>
#include <string>

#include "etap_mla.h"

namespace etaplab_b200 {

// Generic form: Output must be default-constructible with members `o` (a Matrix-like type
// constructible from (rows, cols) with data()) and `l` (a std::vector<double>-like type).
template <class Output, class Problem, class Tiles, class Faults>
Output run_etap(const Problem& p, const Tiles& tiles, const Faults& faults) {
    using MatrixT = decltype(Output{}.o);
    Output out;
    out.o = MatrixT(p.n_q, p.d_v);
    out.l.assign(p.n_q, 0.0);
    const unsigned flags = faults.negate_rescale ? ETAP_FLAG_NEGATE_RESCALE : 0u;
    const int rc = etap_mla_run_etap_f64(
        p.q.data(), static_cast<int64_t>(p.n_q), p.k.data(), static_cast<int64_t>(p.n_kv),
        static_cast<int64_t>(p.d_qk), p.v.data(), static_cast<int64_t>(p.d_v), p.scale,
        static_cast<int64_t>(tiles.b_r), static_cast<int64_t>(tiles.b_c),
        static_cast<int64_t>(tiles.stages), flags, out.o.data(), out.l.data());
    if (rc == ETAP_ERR_SHAPE) throw std::invalid_argument(etap_mla_last_error());
    if (rc != ETAP_OK) throw std::runtime_error(std::string("etap_b200: ") + etap_mla_last_error());
    return out;
}

// Reference-signature form: drop-in for etaplab::run_etap(problem, tiles, hook, faults).
template <class Output, class Problem, class Tiles, class Hook, class Faults>
Output run_etap(const Problem& p, const Tiles& tiles, const Hook& hook, const Faults& faults) {
    if (hook) throw std::invalid_argument("BlockHook is not observable on the GPU path");
    return run_etap<Output>(p, tiles, faults);
}

}  // namespace etaplab_b200
