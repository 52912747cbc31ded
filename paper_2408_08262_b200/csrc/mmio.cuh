// Matrix Market exchange on the host (mmio.cu).
#pragma once

#include <string>
#include <vector>

#include "common.cuh"

namespace airg {

struct MmHost {
  int64_t n = 0, m = 0;
  std::vector<int64_t> rp, ci;
  std::vector<double> v;
};
void mm_read(const std::string& path, MmHost& out);
void mm_write(const std::string& path, int64_t n, int64_t m, const int64_t* rp, const int64_t* ci,
              const double* v);

}  // namespace airg
