// ref_bench_tool.cpp -- TEST INFRASTRUCTURE ONLY. A tiny driver over the
// reference's own bench I/O (proj/core/src/bench.cpp, compiled by path by
// oracle/Makefile) used to produce golden files for the `treedec report`
// compatibility of paper_2408_04093_b200/report.py.
//
//   ref_bench_tool sweep csv|json SEED DTYPE(f64|f32|bf16) HEADS HEAD_DIM N[,N...] NODESxGPUS[,...]
//       run_sweep (bench.cpp:38-116) then write_csv / write_json (bench.cpp:118-147)
//   ref_bench_tool reemit csv|json FILE   parse_bench_file (bench.cpp:273-285), write again
//   ref_bench_tool report FILE            parse_bench_file + write_report (bench.cpp:287-355)
//
// Exit codes: 0 ok, 2 parse / IO error (message "FILE:LINE: message" on stdout,
// the form of `treedec report`, tools/treedec_main.cpp:106-119).
#include "treedec/bench.hpp"

#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace {

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, sep)) out.push_back(item);
    return out;
}

treedec::DType dtype_of(const std::string& s) {
    if (s == "f64") return treedec::DType::Float64;
    if (s == "f32") return treedec::DType::Float32;
    return treedec::DType::Bf16;
}

int parse_or_report(const std::string& path, treedec::SweepOutcome& out) {
    try {
        out = treedec::parse_bench_file(path);
    } catch (const treedec::ParseError& e) {
        std::cout << path << ":" << e.line << ": " << e.message << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cout << e.what() << "\n";
        return 2;
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) return 1;
    const std::string cmd = argv[1];
    if (cmd == "sweep" && argc == 9) {
        treedec::SweepSpec spec;
        spec.seed = std::strtoull(argv[3], nullptr, 10);
        spec.dtype = dtype_of(argv[4]);
        spec.heads = std::atoll(argv[5]);
        spec.head_dim = std::atoll(argv[6]);
        for (const auto& n : split(argv[7], ',')) spec.seq_lens.push_back(std::atoll(n.c_str()));
        for (const auto& c : split(argv[8], ',')) {
            const auto x = split(c, 'x');
            spec.clusters.emplace_back(std::atoi(x[0].c_str()), std::atoi(x[1].c_str()));
        }
        const treedec::SweepOutcome out = treedec::run_sweep(spec);
        if (std::string(argv[2]) == "json") treedec::write_json(out, std::cout);
        else treedec::write_csv(out, std::cout);
        return 0;
    }
    if (cmd == "reemit" && argc == 4) {
        treedec::SweepOutcome out;
        if (int rc = parse_or_report(argv[3], out)) return rc;
        if (std::string(argv[2]) == "json") treedec::write_json(out, std::cout);
        else treedec::write_csv(out, std::cout);
        return 0;
    }
    if (cmd == "report" && argc == 3) {
        treedec::SweepOutcome out;
        if (int rc = parse_or_report(argv[2], out)) return rc;
        treedec::write_report(out, std::cout);
        return 0;
    }
    return 1;
}
