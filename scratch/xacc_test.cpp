#include "../paper_2509_14211_b200/csrc/nbg_internal.hpp"
#include <cstdio>
#include <random>
using namespace nbg;
int main() {
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> U(0, 0.04);
  for (int trial = 0; trial < 5; trial++) {
    unsigned long long L[16] = {0};
    double s = 0; long double ls = 0;
    for (int i = 0; i < 1024; i++) { double v = U(g); host_xacc_add(L, v); s += v; ls += v; }
    printf("%.17g %.17g %.17g\n", xacc_to_double(L), s, (double)ls);
  }
  unsigned long long L[16] = {0};
  host_xacc_add(L, 0.3076171875); printf("%.17g\n", xacc_to_double(L));
  host_xacc_add(L, -1.0); printf("%.17g\n", xacc_to_double(L));
}
namespace nbg { Dist::~Dist() {} }
