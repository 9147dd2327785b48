// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — the reference's own harness driving the GPU path.
// Links the reference's cli.cpp with the `etap_b200` mode patched in (oracle/cli_etap_b200.patch,
// applied by oracle/Makefile to a staged copy; /root/reference is never modified) and calls
// etaplab::cli::cmd_bench / cmd_verify programmatically, as the reference's acceptance.cpp does
// (CLI11 and tools/main.cpp are not needed).
//   harness bench  [seq_lens...]   cmd_bench, modes etap + etap_b200, MLA problems -> CSV on stdout
//   harness verify [tol] [corrupt] cmd_verify with the etap step on the GPU; exit code of cmd_verify
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>

#include "etaplab/cli.hpp"

using namespace etaplab;

int main(int argc, char** argv) {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "bench") {
        cli::BenchOptions o;
        o.modes = {"etap", "etap_b200"};
        o.seq_lens.clear();
        for (int i = 2; i < argc; ++i) o.seq_lens.push_back(std::strtoull(argv[i], nullptr, 10));
        if (o.seq_lens.empty()) o.seq_lens = {1024, 4096};
        o.batch = 2;
        o.heads = 16;
        o.repeats = 5;  // median of 5: the first call of a fresh process also pays CUDA context creation
        o.mla = true;
        o.allow_large = true;
        return cli::cmd_bench(o, std::cout, std::cerr);
    }
    if (cmd == "verify") {
        cli::VerifyOptions o;
        o.etap_impl = "etap_b200";
        o.mla = true;
        o.tolerance = argc > 2 ? std::strtod(argv[2], nullptr) : 1e-4;
        o.corrupt_rescale = argc > 3 && std::strcmp(argv[3], "corrupt") == 0;
        return cli::cmd_verify(o, std::cout, std::cerr);
    }
    std::fprintf(stderr, "usage: harness bench [seq_lens...] | verify [tol] [corrupt]\n");
    return 2;
}
