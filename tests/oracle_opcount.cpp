// oracle_opcount.cpp -- op-counting instantiation of the CPU oracle ("Exact
// flops come from an op-counting instantiation of the oracle RHS: templated on a counting
// scalar type that counts +, -, x, /, fma and exp").
//
// TEST INFRASTRUCTURE (run by tests/test_oracle_opcount.py, which also checks that the
// committed profiles/r2_oracle_opcount.jsonl equals a fresh run): the oracle source is
// compiled unchanged, with its scalar type `double` replaced by the counting type Cnt, so
// every floating-point operation of the oracle's formulation is counted exactly; nothing
// of the CUDA path is involved.  The oracle writes its tensors as full 3x3 index loops
// (symmetric entries computed twice), so these counts are an upper bound of the method's
// flops; SURVEY.md's 22.7k per BSSN RK4 step is the symmetric-packed estimate.
//
// build + run:  g++ -O1 -std=c++17 -I. tests/oracle_opcount.cpp -o /tmp/opcount && /tmp/opcount
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

struct Cnt {
  double v;
  static inline unsigned long long add = 0, mul = 0, dvd = 0, exps = 0, pows = 0, sqrts = 0;
  Cnt() : v(0.0) {}
  Cnt(double x) : v(x) {}
  static void reset() { add = mul = dvd = exps = pows = sqrts = 0; }
};
inline Cnt operator+(Cnt a, Cnt b) { ++Cnt::add; return Cnt(a.v + b.v); }
inline Cnt operator-(Cnt a, Cnt b) { ++Cnt::add; return Cnt(a.v - b.v); }
inline Cnt operator*(Cnt a, Cnt b) { ++Cnt::mul; return Cnt(a.v * b.v); }
inline Cnt operator/(Cnt a, Cnt b) { ++Cnt::dvd; return Cnt(a.v / b.v); }
inline Cnt operator-(Cnt a) { return Cnt(-a.v); }  // sign flip: not a flop
inline Cnt& operator+=(Cnt& a, Cnt b) { a = a + b; return a; }
inline Cnt& operator-=(Cnt& a, Cnt b) { a = a - b; return a; }
inline Cnt& operator*=(Cnt& a, Cnt b) { a = a * b; return a; }
inline Cnt& operator/=(Cnt& a, Cnt b) { a = a / b; return a; }
inline bool operator<(Cnt a, Cnt b) { return a.v < b.v; }
inline bool operator>(Cnt a, Cnt b) { return a.v > b.v; }
inline bool operator<=(Cnt a, Cnt b) { return a.v <= b.v; }
inline bool operator>=(Cnt a, Cnt b) { return a.v >= b.v; }
inline bool operator==(Cnt a, Cnt b) { return a.v == b.v; }
inline bool operator!=(Cnt a, Cnt b) { return a.v != b.v; }
namespace std {
inline Cnt exp(Cnt a) { ++Cnt::exps; return Cnt(std::exp(a.v)); }
inline Cnt pow(Cnt a, Cnt b) { ++Cnt::pows; return Cnt(std::pow(a.v, b.v)); }
inline Cnt sqrt(Cnt a) { ++Cnt::sqrts; return Cnt(std::sqrt(a.v)); }
inline Cnt fabs(Cnt a) { return Cnt(std::fabs(a.v)); }
inline Cnt max(Cnt a, Cnt b) { return a.v < b.v ? b : a; }
inline Cnt min(Cnt a, Cnt b) { return b.v < a.v ? b : a; }
}  // namespace std

#define double Cnt
#include "oracle/chemora_oracle.cpp"
#undef double

namespace {
struct Counts {
  double add, mul, dvd, exps, pows;
  double flops() const { return add + mul + dvd; }  // exp / pow listed separately
};
Counts take(double per) {
  Counts c{Cnt::add / per, Cnt::mul / per, Cnt::dvd / per, Cnt::exps / per, Cnt::pows / per};
  Cnt::reset();
  return c;
}
void print(const char* what, const Counts& c) {
  std::printf("{\"what\": \"%s\", \"add_sub\": %.1f, \"mul\": %.1f, \"div\": %.1f, \"exp\": %.1f, \"pow\": %.1f, "
              "\"flops\": %.1f}\n",
              what, c.add, c.mul, c.dvd, c.exps, c.pows, c.flops());
}
}  // namespace

int main() {
  const int64_t ext[3] = {6, 5, 4};
  const int g = 3;
  const double hs[3] = {0.1, 0.11, 0.12};
  std::vector<Cnt> sp(hs, hs + 3);
  Grid G(ext, g, sp.data());
  const int64_t np = G.npad(), ni = G.nint();
  for (int system : {1, 2}) {
    const int nf = n_gf_of(system);
    // smooth, admissible data: flat BSSN (gt = delta, alpha = 1) plus a small perturbation
    std::vector<Cnt> y(static_cast<size_t>(nf * np)), k(static_cast<size_t>(nf * ni));
    for (int v = 0; v < nf; ++v)
      for (int64_t q = 0; q < np; ++q) {
        double base = 0.0;
        if (system == 2 && (v == 1 || v == 4 || v == 6 || v == 17)) base = 1.0;  // gt_xx, gt_yy, gt_zz, alpha
        y[v * np + q] = Cnt(base + 1e-3 * std::sin(0.37 * (double)q + 1.3 * v));
      }
    std::vector<Cnt> prm(10);
    chemora_oracle_default_bssn_params(prm.data());
    Cnt::reset();
    rhs_any(system, y.data(), k.data(), G, prm.data());
    print(system == 1 ? "wave RHS per point" : "BSSN RHS per point", take((double)ni));
    // one full RK4 step (4 RHS evaluations + the stage combinations), per point
    Cnt dt(1e-3);
    std::vector<Cnt> yy(y);
    chemora_oracle_rk4_order(system, yy.data(), ext, g, sp.data(), dt, 1, prm.data(), 4);
    print(system == 1 ? "wave RK4 step per point" : "BSSN RK4 step per point", take((double)ni));
  }
  return 0;
}
