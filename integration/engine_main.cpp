// integration/engine_main.cpp -- runs the reference simulator (src/sim/engine.cpp,
// unmodified) on a built-in workload and writes its logs, so the same engine can be
// compared with the CPU reference cache/router (oracle build) and with the B200 backend
// (integration/pyg_adapter.cpp): identical event / routing / cache logs = whole-trace
// parity of the hot path.
//
//   engine_<backend> <out_dir> [workflows] [seed]
#include <fstream>
#include <iostream>
#include <string>

#include "pythia/sim/config.hpp"
#include "pythia/sim/engine.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: " << argv[0] << " <out_dir> [workflows] [seed]\n";
    return 2;
  }
  const std::string out = argv[1];
  auto workload = pythia::sim::coding_assistant_workload();
  if (argc > 2) workload.arrivals.total_workflows = std::stoi(argv[2]);
  auto cluster = pythia::sim::coding_assistant_cluster();
  pythia::sim::PolicyConfig policy;
  pythia::sim::SimOptions opt;
  opt.seed = argc > 3 ? std::stoull(argv[3]) : 1;
  opt.record_event_log = true;
  const auto res = pythia::sim::run_simulation(workload, cluster, policy, opt);
  auto dump = [&](const std::string& name, const std::vector<std::string>& lines) {
    std::ofstream f(out + "/" + name);
    for (const auto& l : lines) f << l << "\n";
  };
  dump("event_log.txt", res.event_log);
  dump("routing_log.jsonl", res.routing_log);
  dump("cache_log.jsonl", res.cache_log);
  dump("scale_log.jsonl", res.scale_log);
  std::ofstream(out + "/metrics.json") << res.metrics.to_json().dump(1) << "\n";
  std::cout << "events " << res.event_log.size() << " routes " << res.routing_log.size()
            << " cache " << res.cache_log.size() << "\n";
  return 0;
}
