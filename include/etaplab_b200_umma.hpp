// SPDX-License-Identifier: Apache-2.0
//
// etaplab_b200_umma.hpp — the reference's issued-work model of the two attention GEMMs
// (etaplab::utilization / predicted_speedup, /root/reference/proj/include/etaplab/
// wgmma_model.hpp:64-76, src/wgmma_model.cpp:26-86) restated for the 5th-generation tensor
// core of B200 (tcgen05.mma, cta_group::1, kind::f16), plus the two things the B200 kernel
// adds to the issued work:
//
//   * tile shapes: an MMA instruction is M = 64 or 128 rows (M extents pad to 64; the M = 128
//     form is used whenever 128 rows are available), N pads to 8 for M = 64 and to 16 for
//     M = 128 (minimum 8 / 16), K pads to 16 (bf16);
//   * the hi/lo split of P (DESIGN.md §3 "Numerics"): the PV product of the ETAP mapping is
//     issued with N = 2q (P_hi | P_lo) so bf16 rounding of P does not limit accuracy.
//
// With spec = hopper_wgmma() and pv_passes = 1 the numbers equal the reference's model
// exactly (checked against the compiled reference in tests/test_umma_model_cpu.py). Header
// only, no dependency on the reference's headers; MAC counting only, as in the reference
// (memory traffic, softmax ALU work and barriers are out of model — on B200 the decode is
// HBM-bound, DESIGN.md §3 "Roofline").
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>

namespace etaplab_b200 {

// Same fields and meaning as etaplab::DecodeShape (wgmma_model.hpp:22-29).
struct DecodeShape {
    std::size_t heads = 16;
    std::size_t q_tokens = 1;
    std::size_t kv_len = 4096;
    std::size_t d_qk = 576;
    std::size_t d_v = 512;
    std::size_t batch = 1;
};

enum class ComputeMode { original, etap };

// Instruction-shape rules of one tensor-core generation.
struct UmmaSpec {
    std::size_t m_min = 64;        // M extents pad to a multiple of this
    std::size_t m_wide = 128;      // M form used when >= m_wide rows remain (0: m_min only)
    std::size_t n_step_narrow = 8;   // N granularity with the m_min form
    std::size_t n_step_wide = 16;    // N granularity with the m_wide form
    std::size_t k_step = 16;
    std::size_t pv_passes = 2;     // PV issued for P_hi and P_lo (ETAP mode only)
    double peak_tflops = 1642.0;   // measured dense bf16 on this pool's B200s (MEASURED_PEAKS.json)
};

// The reference's Hopper WGMMA assumptions (wgmma_model.hpp:13-18): m_min 64, n_step 8,
// k_step 16, 148 TFLOP/s, one PV pass.
inline UmmaSpec hopper_wgmma() {
    UmmaSpec s;
    s.m_min = 64;
    s.m_wide = 0;
    s.n_step_narrow = 8;
    s.n_step_wide = 8;
    s.k_step = 16;
    s.pv_passes = 1;
    s.peak_tflops = 148.0;
    return s;
}

// B200 tcgen05 kind::f16, cta_group::1, as the decode kernel issues it.
inline UmmaSpec b200_tcgen05() { return UmmaSpec{}; }

struct GemmPadding {
    std::uint64_t useful_macs = 0;
    std::uint64_t issued_macs = 0;
    std::size_t m_logical = 0;
    std::size_t m_padded = 0;
    double utilization() const { return static_cast<double>(useful_macs) / static_cast<double>(issued_macs); }
    double m_axis_utilization() const {
        return static_cast<double>(m_logical) / static_cast<double>(m_padded);
    }
};

struct UtilizationReport {
    std::uint64_t useful_macs = 0;
    std::uint64_t issued_macs = 0;
    double utilization = 0.0;
    GemmPadding qk;
    GemmPadding pv;
};

namespace detail {
inline std::size_t round_up(std::size_t v, std::size_t step) { return (v + step - 1) / step * step; }

inline void check(const DecodeShape& s, const UmmaSpec& u) {
    if (s.heads < 1 || s.q_tokens < 1 || s.kv_len < 1 || s.d_qk < 1 || s.d_v < 1 || s.batch < 1)
        throw std::invalid_argument("decode shape fields must be >= 1");
    if (u.m_min < 1 || u.n_step_narrow < 1 || u.n_step_wide < 1 || u.k_step < 1 || u.pv_passes < 1)
        throw std::invalid_argument("umma steps must be >= 1");
    if (u.m_wide != 0 && u.m_wide % u.m_min != 0) throw std::invalid_argument("m_wide must be a multiple of m_min");
}

// Issued MACs of an M x N x K product cut into instructions: full m_wide blocks use the wide
// N step, the remaining rows pad to m_min with the narrow N step.
inline GemmPadding count(std::size_t m, std::size_t n, std::size_t k, std::uint64_t batch, std::size_t n_passes,
                         const UmmaSpec& u) {
    GemmPadding g;
    g.m_logical = m;
    g.m_padded = round_up(m, u.m_min);
    const std::uint64_t pk = round_up(k, u.k_step);
    std::uint64_t issued = 0;
    std::size_t rest = g.m_padded;
    if (u.m_wide != 0 && rest >= u.m_wide) {
        const std::size_t wide_rows = rest / u.m_wide * u.m_wide;
        issued += static_cast<std::uint64_t>(wide_rows) * round_up(n * n_passes, u.n_step_wide) * pk;
        rest -= wide_rows;
    }
    issued += static_cast<std::uint64_t>(rest) * round_up(n * n_passes, u.n_step_narrow) * pk;
    g.useful_macs = batch * static_cast<std::uint64_t>(m) * n * k;
    g.issued_macs = batch * issued;
    return g;
}
}  // namespace detail

// Same contract as etaplab::padded_extent (wgmma_model.cpp:43-52) for the narrow form.
enum class GemmAxis { M, N, K };
inline std::size_t padded_extent(std::size_t logical, GemmAxis axis, const UmmaSpec& u) {
    if (logical < 1) throw std::invalid_argument("extent must be >= 1");
    switch (axis) {
        case GemmAxis::M: return detail::round_up(logical, u.m_min);
        case GemmAxis::N: return detail::round_up(logical, u.n_step_narrow);
        case GemmAxis::K: return detail::round_up(logical, u.k_step);
    }
    return logical;
}

// etaplab::utilization (wgmma_model.cpp:54-75): original = query-major (M = folded queries
// for both GEMMs), etap = KV-major (M = kv_len for S^T = K Q^T, M = d_v for O^T = V^T P^T).
inline UtilizationReport utilization(ComputeMode mode, const DecodeShape& s, const UmmaSpec& u = {}) {
    detail::check(s, u);
    const std::size_t q = s.heads * s.q_tokens;
    const std::uint64_t b = s.batch;
    UtilizationReport r;
    if (mode == ComputeMode::original) {
        r.qk = detail::count(q, s.kv_len, s.d_qk, b, 1, u);
        r.pv = detail::count(q, s.d_v, s.kv_len, b, 1, u);
    } else {
        r.qk = detail::count(s.kv_len, q, s.d_qk, b, 1, u);
        r.pv = detail::count(s.d_v, q, s.kv_len, b, u.pv_passes, u);
    }
    r.useful_macs = r.qk.useful_macs + r.pv.useful_macs;
    r.issued_macs = r.qk.issued_macs + r.pv.issued_macs;
    r.utilization = static_cast<double>(r.useful_macs) / static_cast<double>(r.issued_macs);
    return r;
}

// etaplab::predicted_speedup (wgmma_model.cpp:77-86): issued(original) / (issued(etap) +
// one transpose of d_v * q per batch element). An issued-work bound, not a wall-clock one.
inline double predicted_speedup(const DecodeShape& s, const UmmaSpec& u = {}) {
    const UtilizationReport o = utilization(ComputeMode::original, s, u);
    const UtilizationReport e = utilization(ComputeMode::etap, s, u);
    const double transpose = static_cast<double>(s.batch) * static_cast<double>(s.d_v) *
                             static_cast<double>(s.heads * s.q_tokens);
    return static_cast<double>(o.issued_macs) / (static_cast<double>(e.issued_macs) + transpose);
}

// Tensor-core time of the issued work at the spec's peak (µs): 2 flops per MAC.
inline double tensor_time_us(const UtilizationReport& r, const UmmaSpec& u) {
    return 2.0 * static_cast<double>(r.issued_macs) / (u.peak_tflops * 1e6);
}

}  // namespace etaplab_b200
