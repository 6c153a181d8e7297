// TEST INFRASTRUCTURE (oracle): how nlohmann::json 3.11.3 (the reference's
// JSON library, bench/config.hpp:8) prints doubles -- "<bits hex> <dump>" per
// line for a seeded mix of raw bit patterns, unit-range values and
// float-valued decimals. Pins paper_1910_02270_b200/outputs.py's Grisu2
// printer (tests/golden/nlohmann_doubles.txt, tests/test_outputs.py).
#include <cmath>
#include <cstdlib>
#include <json.hpp>
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <random>
int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 4000;
  std::mt19937_64 g(7);
  for (int i = 0; i < n; ++i) {
    uint64_t b = g();
    double d;
    if (i % 3 == 0) { std::memcpy(&d, &b, 8); }
    else if (i % 3 == 1) { d = std::ldexp((double)(b >> 11) / 9007199254740992.0, (int)(g() % 80) - 40); }
    else { d = (double)(float)((double)(b >> 40) / (double)(1ull << 24) * std::pow(10.0, (int)(g() % 30) - 15)); }
    nlohmann::json x = d;
    std::printf("%016llx %s\n", (unsigned long long)[&]{uint64_t u; std::memcpy(&u,&d,8); return u;}(), x.dump().c_str());
  }
}
