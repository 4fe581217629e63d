// oracle/cmd_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Minimal stand-in for the reference CLI (tools/main.cpp needs CLI11, absent here):
//   cmd_driver <command> <config.json> <out_dir> [threads]
// calls dfs::cli::run_command (commands.cpp:735). oracle/Makefile links it twice:
// cmd_ref against the reference's own hot-path sources, cmd_gpu against the B200
// drop-in library, so tests can compare the two runs' report.csv and masks/*.dfsm
// byte for byte.
#include <cstdio>
#include <exception>
#include <fstream>

#include <json.hpp>

#include "dfs/commands.hpp"

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s <command> <config.json> <out_dir> [threads]\n", argv[0]);
    return 2;
  }
  try {
    std::ifstream in(argv[2]);
    const nlohmann::json config = nlohmann::json::parse(in);
    return dfs::cli::run_command(argv[1], config, argv[3], argc > 4 ? std::atoi(argv[4]) : 0);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
