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
#include <vector>
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

    // precision: only exact64 storage maps to the GPU's bf16 x bf16 -> fp32 (Precision,
    // matrix.hpp:22); fp32 / fp16emu problems raise std::invalid_argument, not a silent bf16 run
    int prec_mirrored = 0;
    for (Precision pr : {Precision::fp32, Precision::fp16emu}) {
        AttentionProblem pp = mla_problem(3, 16, 128);
        pp.precision = pr;
        try {
            etaplab_b200::run_etap<AttentionOutput>(pp, TileConfig{}, EtapFaults{});
        } catch (const std::invalid_argument&) {
            ++prec_mirrored;
        }
    }
    std::printf("{\"precision_rejected\": %d}\n", prec_mirrored);

    // BlockHook through the adapter against the reference's OWN hook stream (run_etap with a
    // recording hook on the same problem): same call count and order (query blocks of b_r rows
    // outer, KV blocks of b_c rows inner, etap.cpp:115-129), same vector lengths, m / l /
    // rescale equal within fp32 accuracy; plus the rules of the reference's StateChecker
    // (cli.cpp:43-70: m never decreases, l > 0, rescale 0 on first touch else in (0, 1]). The
    // negate_rescale fault (EtapFaults, etap.hpp:39-41, etap.cpp:62) flips the factor applied to
    // the accumulator, not the reported state: as in the reference, the invariants still hold
    // and the fault shows in the output (the verifier's equivalence check, cli.cpp:147-160).
    struct Step {
        std::size_t qb, kb;
        std::vector<double> m_old, m, l, rescale;
    };
    auto record = [](std::vector<Step>& v) {
        return BlockHook([&v](const BlockStepInfo& info) {
            v.push_back(Step{info.query_block, info.kv_block, info.m_old, info.state.m, info.state.l, info.rescale});
        });
    };
    int hook_ok = 0, hook_cases = 0;
    const std::size_t hcases[][4] = {{32, 1000, 64, 64}, {32, 1000, 16, 128}, {20, 777, 16, 100}, {16, 300, 8, 16}};
    for (auto& hc : hcases) {
        for (int fault = 0; fault < 2; ++fault) {
            ++hook_cases;
            const AttentionProblem hp = mla_problem(7, hc[0], hc[1]);
            const TileConfig tc{hc[2], hc[3], 2};
            std::vector<Step> ref_steps, gpu_steps;
            run_etap(hp, tc, record(ref_steps));
            EtapFaults faults{};
            faults.negate_rescale = fault != 0;
            const AttentionOutput g = etaplab_b200::run_etap<AttentionOutput>(hp, tc, record(gpu_steps), faults);
            std::size_t violations = 0;
            double dm = 0, dl = 0, dr = 0;
            bool same_shape = ref_steps.size() == gpu_steps.size();
            for (std::size_t s = 0; same_shape && s < ref_steps.size(); ++s) {
                const Step &a = ref_steps[s], &b = gpu_steps[s];
                if (a.qb != b.qb || a.kb != b.kb || a.m.size() != b.m.size()) { same_shape = false; break; }
                for (std::size_t i = 0; i < a.m.size(); ++i) {
                    const bool first_touch = std::isinf(b.m_old[i]) && b.m_old[i] < 0;
                    if (b.m[i] < b.m_old[i] || !(b.l[i] > 0.0) ||
                        (first_touch ? b.rescale[i] != 0.0 : !(b.rescale[i] > 0.0 && b.rescale[i] <= 1.0)))
                        ++violations;
                    dm = std::max(dm, std::fabs(a.m[i] - b.m[i]));
                    dl = std::max(dl, std::fabs(a.l[i] - b.l[i]) / a.l[i]);
                    dr = std::max(dr, std::fabs(a.rescale[i] - b.rescale[i]));
                }
            }
            const double e = rmse(g.o, attention_ref(hp).o);
            const bool ok = same_shape && violations == 0 && dm <= 1e-4 && dl <= 1e-4 && dr <= 1e-4 &&
                            (fault ? e > 100 * 2e-5 : e <= 2e-5);
            hook_ok += ok;
            std::printf("{\"block_hook\": {\"n_q\": %zu, \"n_kv\": %zu, \"b_r\": %zu, \"b_c\": %zu, \"negate_rescale\": %s, "
                        "\"calls\": %zu, \"reference_calls\": %zu, \"same_order\": %s, \"violations\": %zu, "
                        "\"max_abs_dm\": %.2e, \"max_rel_dl\": %.2e, \"max_abs_drescale\": %.2e, \"rmse\": %.3e, "
                        "\"ok\": %s}}\n",
                        hc[0], hc[1], hc[2], hc[3], fault ? "true" : "false", gpu_steps.size(), ref_steps.size(),
                        same_shape ? "true" : "false", violations, dm, dl, dr, e, ok ? "true" : "false");
        }
    }
    return (failures == 0 && mirrored == 2 && prec_mirrored == 2 && hook_ok == hook_cases) ? 0 : 1;
}
