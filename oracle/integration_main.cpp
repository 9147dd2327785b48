// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — integration check of the drop-in boundary.
// Builds problems with the UNMODIFIED reference library (etaplab::make_problem, with the MLA
// aliasing V = K.col_block(0, 512)), then runs
//   * etaplab::attention_ref            (the reference oracle, attention.cpp:44-77)
//   * etaplab::run_etap                 (the reference hot path, etap.cpp:102-148)
//   * etaplab_b200::run_etap<...>       (include/etaplab_b200.hpp -> libetap_mla.so, the GPU)
// on the same operands and prints one JSON line per case. Exit 0 iff every GPU RMSE <= 2e-5
// and the reference error behaviour (std::invalid_argument) is mirrored.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "etaplab/attention.hpp"
#include "etaplab/etap.hpp"
#include "etaplab/matrix.hpp"
#include "etaplab/tiled_standard.hpp"
#include "etaplab_b200.hpp"

using namespace etaplab;

static AttentionProblem mla_problem(std::uint64_t seed, std::size_t heads, std::size_t ctx) {
    // reference generator (matrix.cpp:153-165), seeds as in attention.cpp:38-39; bf16 rounding
    // is applied by the adapter on the way in, so round here too so the oracle sees the same
    // operands the GPU sees
    Matrix q = matrix_from_seed(heads, 576, seed * 3 + 1, Dist::normal);
    Matrix kv = matrix_from_seed(ctx, 576, seed * 3 + 2, Dist::normal);
    auto bf16 = [](Matrix& m) {
        for (std::size_t i = 0; i < m.size(); ++i) {
            float f = static_cast<float>(m.data()[i]);
            // exact binary64 -> bf16 RNE: via frexp/ldexp (single rounding)
            const double ax = std::fabs(m.data()[i]);
            if (ax != 0.0) {
                int e;
                std::frexp(ax, &e);
                const double r = std::nearbyint(std::ldexp(ax, 8 - e));
                f = static_cast<float>(std::copysign(std::ldexp(r, e - 8), m.data()[i]));
            }
            m.data()[i] = f;
        }
    };
    bf16(q);
    bf16(kv);
    Matrix v = kv.col_block(0, 512);
    return make_problem(q, kv, v, 1.0 / 24.0, Precision::exact64);
}

int main() {
    int failures = 0;
    const std::size_t cases[][2] = {{16, 1024}, {16, 257}, {5, 77}, {32, 4096}};
    for (auto& c : cases) {
        const AttentionProblem p = mla_problem(42, c[0], c[1]);
        const TileConfig tiles{64, 64, 2};
        const AttentionOutput ref = attention_ref(p);
        auto t0 = std::chrono::steady_clock::now();
        const AttentionOutput cpu = run_etap(p, tiles);
        auto t1 = std::chrono::steady_clock::now();
        AttentionOutput gpu;
        try {
            gpu = etaplab_b200::run_etap<AttentionOutput>(p, tiles, BlockHook{}, EtapFaults{});
        } catch (const std::exception& e) {
            std::printf("{\"case\": [%zu, %zu], \"error\": \"%s\"}\n", c[0], c[1], e.what());
            return 2;
        }
        auto t2 = std::chrono::steady_clock::now();
        const double e_gpu = rmse(gpu.o, ref.o), e_cpu = rmse(cpu.o, ref.o);
        double l_err = 0.0;
        for (std::size_t i = 0; i < p.n_q; ++i) l_err = std::max(l_err, std::fabs(gpu.l[i] - ref.l[i]));
        const bool ok = e_gpu <= 2e-5 && l_err <= 1e-4;
        failures += !ok;
        std::printf("{\"case\": {\"n_q\": %zu, \"n_kv\": %zu}, \"rmse_gpu_vs_attention_ref\": %.3e, "
                    "\"rmse_cpu_run_etap_vs_attention_ref\": %.3e, \"lse_maxabs\": %.3e, "
                    "\"cpu_run_etap_ms\": %.3f, \"gpu_run_etap_ms_incl_h2d_d2h\": %.3f, \"ok\": %s}\n",
                    c[0], c[1], e_gpu, e_cpu, l_err,
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count(), ok ? "true" : "false");
    }
    // error behaviour: tile fields < 1 and an independent V both raise std::invalid_argument
    const AttentionProblem p = mla_problem(1, 16, 64);
    int mirrored = 0;
    try {
        etaplab_b200::run_etap<AttentionOutput>(p, TileConfig{16, 0, 2}, EtapFaults{});
    } catch (const std::invalid_argument&) {
        ++mirrored;
    }
    try {
        etaplab_b200::run_etap<AttentionOutput>(make_problem(42, 16, 64, 576, 512), TileConfig{}, EtapFaults{});
    } catch (const std::invalid_argument&) {
        ++mirrored;
    }
    std::printf("{\"invalid_argument_mirrored\": %d}\n", mirrored);

    // BlockHook through the adapter: the GPU's per-tile softmax state replayed into the
    // reference's own observer type, checked with the rules of the reference's StateChecker
    // (cli.cpp:43-70: m never decreases, l > 0, rescale 0 on first touch else in (0, 1]). The
    // negate_rescale fault (EtapFaults, etap.hpp:39-41, etap.cpp:62) flips the factor applied to
    // the accumulator, not the reported state: as in the reference, the invariants still hold
    // and the fault shows in the output (the verifier's equivalence check, cli.cpp:147-160).
    int hook_ok = 0;
    for (int fault = 0; fault < 2; ++fault) {
        const AttentionProblem hp = mla_problem(7, 32, 1000);
        std::size_t calls = 0, violations = 0;
        BlockHook hook = [&](const BlockStepInfo& info) {
            ++calls;
            for (std::size_t i = 0; i < info.m_old.size(); ++i) {
                const bool first_touch = std::isinf(info.m_old[i]) && info.m_old[i] < 0;
                if (info.state.m[i] < info.m_old[i]) ++violations;
                else if (!(info.state.l[i] > 0.0)) ++violations;
                else if (first_touch ? info.rescale[i] != 0.0 : !(info.rescale[i] > 0.0 && info.rescale[i] <= 1.0))
                    ++violations;
            }
        };
        EtapFaults faults{};
        faults.negate_rescale = fault != 0;
        const AttentionOutput g = etaplab_b200::run_etap<AttentionOutput>(hp, TileConfig{64, 64, 2}, hook, faults);
        const double e = rmse(g.o, attention_ref(hp).o);
        const std::size_t want = ((hp.n_q + 15) / 16) * ((hp.n_kv + 63) / 64);
        const bool ok = violations == 0 && calls == want && (fault ? e > 100 * 2e-5 : e <= 2e-5);
        hook_ok += ok;
        std::printf("{\"block_hook\": {\"negate_rescale\": %s, \"calls\": %zu, \"expected_calls\": %zu, "
                    "\"violations\": %zu, \"rmse\": %.3e, \"ok\": %s}}\n", fault ? "true" : "false", calls, want,
                    violations, e, ok ? "true" : "false");
    }
    return (failures == 0 && mirrored == 2 && hook_ok == 2) ? 0 : 1;
}
