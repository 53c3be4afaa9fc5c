// Host-side drop-in modules (io.hpp, perf_model.hpp, theory.hpp) driven from
// tests/test_host_modules.py, which compares every output with the reference
// build (oracle/_ref/libbkref.so).  No GPU is touched.
//   test_host mm <in> <out>          read Matrix Market, write it back
//   test_host bv <in> <out>          read a block-vector file, write it back
//   test_host spectrum <in.mtx>      eigenvalues, one %.17g per line
//   test_host rate <0|1> <p> <q> <ev...>   rate_classical(p) / rate_global(p, q)
//   test_host chars <kernel> <n> <k> <p> <z>   omega beta tau
// Exit codes: 0 ok, 1 IoError, 2 other blockkrylov error.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "blockkrylov/io.hpp"
#include "blockkrylov/perf_model.hpp"
#include "blockkrylov/theory.hpp"

namespace bk = blockkrylov;

int main(int argc, char** argv) {
  if (argc < 2) return 64;
  const std::string cmd = argv[1];
  try {
    if (cmd == "mm" && argc == 4) {
      bk::save_matrix_market(argv[3], bk::load_matrix_market(argv[2]));
    } else if (cmd == "bv" && argc == 4) {
      bk::save_block_vector(argv[3], bk::load_block_vector(argv[2]));
    } else if (cmd == "spectrum" && argc == 3) {
      const bk::Spectrum s = bk::spectrum_of(bk::load_matrix_market(argv[2]));
      for (double v : s.values()) std::printf("%.17g\n", v);
    } else if (cmd == "rate" && argc >= 5) {
      std::vector<double> ev;
      for (int i = 5; i < argc; ++i) ev.push_back(std::strtod(argv[i], nullptr));
      const bk::Spectrum s(ev);
      const std::size_t p = std::strtoull(argv[3], nullptr, 10), q = std::strtoull(argv[4], nullptr, 10);
      std::printf("%.17g\n", argv[2][0] == '1' ? bk::rate_global(s, p, q) : bk::rate_classical(s, p));
    } else if (cmd == "chars" && argc == 7) {
      const auto c = bk::characteristics(bk::parse_kernel(argv[2]), std::strtoull(argv[3], nullptr, 10),
                                         std::strtoull(argv[4], nullptr, 10),
                                         std::strtoull(argv[5], nullptr, 10),
                                         std::strtoull(argv[6], nullptr, 10));
      std::printf("%llu %llu %llu\n", (unsigned long long)c.omega, (unsigned long long)c.beta,
                  (unsigned long long)c.tau);
    } else {
      return 64;
    }
  } catch (const bk::IoError& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  } catch (const bk::Error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  }
  return 0;
}
