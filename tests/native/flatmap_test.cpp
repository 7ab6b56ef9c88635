// Randomised check of sgf::FlatMap (runtime.h) against std::unordered_map:
// inserts, overwrites, erases (backward-shift deletion), lookups, iteration.
#include <cstdio>
#include <random>
#include <unordered_map>

#include "runtime.h"

int main() {
  std::mt19937_64 rng(7);
  for (int round = 0; round < 20; ++round) {
    sgf::FlatMap<long long> fm(round % 3 == 0 ? 1 : 1000);
    std::unordered_map<uint64_t, long long> ref;
    const int universe = 50 + round * 300;
    for (int op = 0; op < 20000; ++op) {
      const uint64_t k = sgf::bkey((int)(rng() % universe), (int)(rng() % universe));
      const int what = (int)(rng() % 10);
      if (what < 5) {
        const long long v = (long long)(rng() % 1000000);
        fm[k] = v;
        ref[k] = v;
      } else if (what < 8) {
        const bool a = fm.erase(k), b = ref.erase(k) > 0;
        if (a != b) { std::printf("erase mismatch\n"); return 1; }
      } else {
        const long long* p = fm.find(k);
        auto it = ref.find(k);
        if ((p == nullptr) != (it == ref.end()) || (p && *p != it->second)) {
          std::printf("find mismatch\n");
          return 1;
        }
      }
      if (fm.size() != ref.size()) { std::printf("size mismatch\n"); return 1; }
    }
    size_t seen = 0;
    bool ok = true;
    fm.for_each([&](uint64_t k, long long& v) {
      ++seen;
      auto it = ref.find(k);
      if (it == ref.end() || it->second != v) ok = false;
    });
    if (!ok || seen != ref.size()) { std::printf("iteration mismatch\n"); return 1; }
  }
  std::printf("ok\n");
  return 0;
}
