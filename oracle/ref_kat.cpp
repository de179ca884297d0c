// ORACLE — TEST INFRASTRUCTURE ONLY.
// Known-answer generator compiled against the reference's own header
// (/root/reference/proj/include/fj/value.hpp, used in place, never copied):
// prints fj::TupleHash (value.hpp:61-67) of integer tuples read from stdin,
// one tuple per line ("n v1 ... vn"), as "0x%016llx". Built by
// oracle/build_ref.sh into oracle/_ref/ref_kat.
#include <cstdint>
#include <cstdio>
#include <iostream>

#include "fj/value.hpp"

int main() {
  int n;
  while (std::cin >> n) {
    fj::Tuple t;
    for (int i = 0; i < n; ++i) {
      long long v;
      std::cin >> v;
      t.push_back(fj::Value(static_cast<std::int64_t>(v)));
    }
    std::printf("0x%016llx\n", static_cast<unsigned long long>(fj::TupleHash{}(t)));
  }
  return 0;
}
