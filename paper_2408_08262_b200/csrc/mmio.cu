// Matrix Market exchange (reference: matrix_market.hpp:11-19,
// matrix_market.cpp:27-81): "coordinate real general", 1-based indices,
// duplicates summed, values written with 17 significant digits so a round
// trip is exact. Host-only code: the file is read in one block and tokenised
// in place; entries are assembled exactly like SparseMatrix::from_triplets
// (sparse.cpp:48-80) -- an (unstable) std::sort by (row, col) of the entry
// list in file order, then each run of equal keys summed left to right -- so
// the stored values, duplicates included, match the reference's bit for bit
// (same library sort, same input sequence, same comparisons).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "mmio.cuh"

namespace airg {

namespace {

[[noreturn]] void fail(const std::string& path, const std::string& msg) {
  throw RuntimeError("matrix market: " + path + ": " + msg);
}

std::string lower(std::string s) {
  for (char& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

struct Entry {  // the reference's Triplet layout: row, col, value
  int64_t row, col;
  double value;
};

// whitespace-separated token reader over the file buffer (istream >> style)
struct Tokens {
  const char* p;
  const char* end;
  bool next_int(int64_t& out) {
    skip();
    if (p >= end) return false;
    char* q = nullptr;
    errno = 0;
    const long long v = std::strtoll(p, &q, 10);
    if (q == p || errno == ERANGE) return false;
    p = q;
    out = v;
    return true;
  }
  bool next_double(double& out) {
    skip();
    if (p >= end) return false;
    char* q = nullptr;
    const double v = std::strtod(p, &q);
    if (q == p) return false;
    p = q;
    out = v;
    return true;
  }
  void skip() {
    while (p < end && std::isspace((unsigned char)*p)) ++p;
  }
};

}  // namespace

void mm_read(const std::string& path, MmHost& out) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(path, "cannot open for reading");
  std::string buf;
  {
    char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.append(chunk, got);
    std::fclose(f);
  }
  const char* p = buf.data();
  const char* end = p + buf.size();
  auto getline = [&](std::string& line) {
    if (p >= end) return false;
    const char* nl = p;
    while (nl < end && *nl != '\n') ++nl;
    line.assign(p, nl);
    if (!line.empty() && line.back() == '\r') line.pop_back();
    p = nl < end ? nl + 1 : end;
    return true;
  };
  std::string line;
  if (!getline(line)) fail(path, "empty file");
  {
    Tokens t{line.data(), line.data() + line.size()};
    std::string tok[5];
    for (auto& s : tok) {
      t.skip();
      const char* b = t.p;
      while (t.p < t.end && !std::isspace((unsigned char)*t.p)) ++t.p;
      s.assign(b, t.p);
    }
    if (tok[0] != "%%MatrixMarket" || lower(tok[1]) != "matrix") fail(path, "malformed header: " + line);
    if (lower(tok[2]) != "coordinate" || lower(tok[3]) != "real" || lower(tok[4]) != "general")
      fail(path, "unsupported format (need coordinate real general): " + line);
  }
  // comments and blank lines, then the size line
  bool have = false;
  while (getline(line))
    if (!line.empty() && line[0] != '%') {
      have = true;
      break;
    }
  if (!have) line.clear();
  int64_t n = 0, m = 0, nnz = 0;
  {
    Tokens t{line.data(), line.data() + line.size()};
    if (!t.next_int(n) || !t.next_int(m) || !t.next_int(nnz) || n < 0 || m < 0 || nnz < 0)
      fail(path, "malformed size line: " + line);
  }
  std::vector<Entry> e;
  e.reserve((size_t)nnz);
  Tokens t{p, end};
  for (int64_t k = 0; k < nnz; ++k) {
    int64_t i, j;
    double v;
    if (!t.next_int(i) || !t.next_int(j) || !t.next_double(v)) fail(path, "truncated entry list");
    if (i < 1 || i > n || j < 1 || j > m) fail(path, "index out of bounds at entry " + std::to_string(k + 1));
    e.push_back({i - 1, j - 1, v});
  }
  std::sort(e.begin(), e.end(),
            [](const Entry& a, const Entry& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
  out.n = n;
  out.m = m;
  out.rp.assign((size_t)n + 1, 0);
  out.ci.clear();
  out.v.clear();
  out.ci.reserve(e.size());
  out.v.reserve(e.size());
  size_t k = 0;
  for (int64_t r = 0; r < n; ++r) {
    while (k < e.size() && e[k].row == r) {
      const int64_t c = e[k].col;
      double s = e[k].value;
      for (++k; k < e.size() && e[k].row == r && e[k].col == c; ++k) s += e[k].value;
      out.ci.push_back(c);
      out.v.push_back(s);
    }
    out.rp[(size_t)r + 1] = (int64_t)out.ci.size();
  }
}

void mm_write(const std::string& path, int64_t n, int64_t m, const int64_t* rp, const int64_t* ci,
              const double* v) {
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) fail(path, "cannot open for writing");
  std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
  std::fprintf(f, "%lld %lld %lld\n", (long long)n, (long long)m, (long long)(n ? rp[n] : 0));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      std::fprintf(f, "%lld %lld %.17g\n", (long long)(i + 1), (long long)(ci[k] + 1), v[k]);
  if (std::fclose(f) != 0) fail(path, "write failed on close");
}

}  // namespace airg
