// cli_main.cpp -- TEST INFRASTRUCTURE ONLY: the end-to-end parity harness of
// SURVEY.md 8(b).  A main() around the reference's own command functions
// (/root/reference/proj/src/cli.cpp: cmd_eval, cmd_slice, cmd_ccmap,
// cmd_gen_dict, cmd_noise -- compiled from the reference sources in place by
// oracle/Makefile, never copied), linked twice:
//   oracle/_ref/cli_ref  -- against the reference library itself;
//   oracle/_ref/cli_b200 -- against the drop-in (-I include/mrf_b200, whose
//                           mrf/*.hpp shims resolve the library headers, and
//                           libmrf_b200.so + libmrfg.so on the GPU).
// tests/test_cli_harness.py runs both on the same command and diffs the CSVs.
// Usage: cli_{ref,b200} <eval|slice|ccmap|gen-dict|noise|gen-schedule> <out_dir> [key=value ...]
#include <cstdio>
#include <exception>
#include <string>

#include "mrf/cli.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <command> <out_dir> [key=value ...]\n", argv[0]);
        return 2;
    }
    try {
        mrf::RunConfig cfg;
        cfg.out_dir = argv[2];
        for (int i = 3; i < argc; ++i) mrf::apply_override(cfg, argv[i]);
        const std::string cmd = argv[1];
        if (cmd == "eval") return mrf::cmd_eval(cfg);
        if (cmd == "slice") return mrf::cmd_slice(cfg);
        if (cmd == "ccmap") return mrf::cmd_ccmap(cfg);
        if (cmd == "gen-dict") return mrf::cmd_gen_dict(cfg);
        if (cmd == "noise") return mrf::cmd_noise(cfg);
        if (cmd == "gen-schedule") return mrf::cmd_gen_schedule(cfg);
        std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
