// config_tool.cpp -- drives the C++ mirror's RunConfig (include/solkin_b200_config.hpp)
// for tests/test_config.py, which compares its output with the reference's
// RunConfig (oracle/_ref, config.cpp) on the same inputs.
//
//   config_tool eval <preset|-> <file|-> <resolve 0|1> [key value]...
//       -> "ok\n" echo "--\n" violations (one per line) "--\n" nsteps
//       -> "error\n" message
//   config_tool matrices <alpha> <order>   -> the `solkin matrices` table
//   config_tool layered <file|-> <preset|-> <limiter|-> <out|-> <threads>
//       -> resolve_run_config (cmd_run's layering + validate), as eval
//   config_tool run <file|-> <preset|->   -> `solkin run` on the device (GPU only)
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>

#include "solkin_b200_config.hpp"

using solkin_b200::RunConfig;

static std::string arg(const char* s) { return std::string(s) == "-" ? "" : s; }

static void report(const RunConfig& c) {
    std::cout << "ok\n" << c.echo() << "--\n";
    for (const auto& v : c.violations()) std::cout << v << "\n";
    std::cout << "--\n" << c.nsteps() << "\n";
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string cmd = argv[1];
    try {
        if (cmd == "eval" && argc >= 5) {
            RunConfig c;
            if (!arg(argv[2]).empty()) c = RunConfig::preset(argv[2]);
            if (!arg(argv[3]).empty()) c.apply_file(argv[3]);
            for (int i = 5; i + 1 < argc; i += 2) c.apply_kv(argv[i], argv[i + 1]);
            if (std::atoi(argv[4])) c.resolve();
            report(c);
            return 0;
        }
        if (cmd == "layered" && argc == 7) {
            report(solkin_b200::resolve_run_config(arg(argv[2]), arg(argv[3]), arg(argv[4]),
                                                   arg(argv[5]), std::atoi(argv[6])));
            return 0;
        }
        if (cmd == "run" && argc == 4) {
            const RunConfig cfg = solkin_b200::resolve_run_config(arg(argv[2]), arg(argv[3]));
            const sk_run_result r = solkin_b200::run(cfg);
            std::cout << "exit " << r.exit_code << " steps " << r.steps_done << "\n";
            return 0;
        }
        if (cmd == "matrices" && argc == 4) {
            std::cout << solkin_b200::matrices_text(std::strtod(argv[2], nullptr), std::atoi(argv[3]));
            return 0;
        }
    } catch (const std::exception& e) {
        std::cout << "error\n" << e.what();
        return 0;
    }
    return 2;
}
