// TEST INFRASTRUCTURE (golden generator, run here where /root/reference
// exists; the outputs are committed under tests/golden/seq_ref/):
// the reference's own IO surface on a small generated sequence --
// cmd_gen (generate_systems + save_sequence: manifest.json, Matrix Market
// blocks, vector JSON), cmd_solve (solve.csv + run_manifest.json) and
// cmd_sweep_gamma (sweep.csv) -- so the GPU path's IO module can be checked
// for byte-compatible files (proj/core/src/driver.cpp:131-279,
// manifest.cpp, matrix_market.cpp; docs/formats.md).
#include <filesystem>
#include <iostream>
#include <vector>

#include "hkkt/driver.hpp"
#include "hkkt/generator.hpp"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::filesystem::path out = argv[1];
  hkkt::GeneratorSpec spec;
  spec.n_x = 60;
  spec.m_c = 15;
  spec.m_d = 12;
  spec.sequence_length = 3;
  spec.seed = 41;
  int rc = hkkt::cmd_gen(spec, out / "seq", std::cerr);
  if (rc != 0) return rc;
  hkkt::SolverConfig cfg;
  rc = hkkt::cmd_solve(out / "seq" / "manifest.json", cfg, out / "solve", std::cerr);
  std::cout << "solve rc " << rc << "\n";
  const std::vector<double> gammas{1e2, 1e4, 1e6};
  rc = hkkt::cmd_sweep_gamma(out / "seq" / "manifest.json", gammas, cfg, out / "sweep", std::cerr);
  std::cout << "sweep rc " << rc << "\n";
  return 0;
}
