// SPDX-License-Identifier: Apache-2.0
// etap_model — the reference's `etaplab model` report (cmd_model, /root/reference/proj/src/
// cli.cpp:308-343: issued vs useful MACs of the original and ETAP mappings, predicted
// speedup) for the B200 tensor core, from include/etaplab_b200_umma.hpp.
//
//   etap_model [--spec b200|hopper] [--heads 16] [--q-tokens 1] [--batch 1]
//              [--kv 512,1024,...] [--d-qk 576] [--d-v 512] [--peak-tflops X]
// CSV on stdout with the reference's columns plus spec fields and tensor_time_us.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/etaplab_b200_umma.hpp"

using namespace etaplab_b200;

int main(int argc, char** argv) {
    UmmaSpec spec = b200_tcgen05();
    DecodeShape shape;
    std::vector<std::size_t> kvs = {512, 1024, 2048, 4096, 8192, 16384, 32768, 65536};
    double peak = -1.0;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) { std::fprintf(stderr, "missing value for %s\n", a.c_str()); std::exit(2); }
            return argv[++i];
        };
        if (a == "--spec") {
            const std::string v = val();
            if (v == "hopper") spec = hopper_wgmma();
            else if (v == "b200") spec = b200_tcgen05();
            else { std::fprintf(stderr, "unknown spec %s\n", v.c_str()); return 2; }
        } else if (a == "--heads") shape.heads = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--q-tokens") shape.q_tokens = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--batch") shape.batch = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--d-qk") shape.d_qk = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--d-v") shape.d_v = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--peak-tflops") peak = std::atof(val().c_str());
        else if (a == "--kv") {
            kvs.clear();
            std::stringstream ss(val());
            std::string tok;
            while (std::getline(ss, tok, ',')) kvs.push_back(std::strtoull(tok.c_str(), nullptr, 10));
        } else {
            std::fprintf(stderr, "unknown option %s\n", a.c_str());
            return 2;
        }
    }
    if (peak > 0) spec.peak_tflops = peak;
    if (kvs.empty()) { std::fprintf(stderr, "model: kv length list is empty\n"); return 2; }
    std::printf("mode,heads,q_tokens,batch,kv_len,d_qk,d_v,m_min,m_wide,n_step_narrow,n_step_wide,k_step,"
                "pv_passes,useful_macs,issued_macs,utilization,qk_m_axis_utilization,pv_m_axis_utilization,"
                "predicted_speedup,effective_tflops,tensor_time_us\n");
    try {
        for (std::size_t kv : kvs) {
            shape.kv_len = kv;
            const double sp = predicted_speedup(shape, spec);
            for (ComputeMode m : {ComputeMode::original, ComputeMode::etap}) {
                const UtilizationReport r = utilization(m, shape, spec);
                std::printf("%s,%zu,%zu,%zu,%zu,%zu,%zu,%zu,%zu,%zu,%zu,%zu,%zu,%llu,%llu,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g\n",
                            m == ComputeMode::original ? "original" : "etap", shape.heads, shape.q_tokens,
                            shape.batch, kv, shape.d_qk, shape.d_v, spec.m_min, spec.m_wide, spec.n_step_narrow,
                            spec.n_step_wide, spec.k_step, m == ComputeMode::etap ? spec.pv_passes : 1,
                            static_cast<unsigned long long>(r.useful_macs),
                            static_cast<unsigned long long>(r.issued_macs), r.utilization,
                            r.qk.m_axis_utilization(), r.pv.m_axis_utilization(), sp,
                            spec.peak_tflops * r.utilization, tensor_time_us(r, spec));
            }
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "model: %s\n", e.what());
        return 2;
    }
    return 0;
}
