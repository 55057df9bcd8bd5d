// io.cu — the input path of SURVEY.md §8(f) rank 2 (io.hpp:68-250):
//   * Matrix Market coordinate and SNAP edge-list readers, Matrix Market
//     writer (host text parsing, same acceptance rules and DataError cases
//     as the reference);
//   * graph Laplacian and symmetrization on the device, bit-identical to
//     the reference's sequential sums: a stable radix sort groups the
//     triplets by row (Laplacian degrees) or by unordered pair
//     (symmetrize), so each group keeps the input order, and one thread
//     folds its group from 0.0 in that order, as io.hpp:215-220 / :233-237
//     do with their vector / std::map accumulators.
#include <cub/cub.cuh>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "common.cuh"

namespace pmmf_b200 {

int guarded_call(char* err, size_t errlen, void (*fn)(void*), void* ctx);

namespace {

constexpr int kThreads = 256;

// ------------------------------------------------------------ host text
std::string lowered(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// whitespace tokens of a line (what `istream >> std::string` yields)
void split(const std::string& line, std::vector<std::string_view>& out) {
  out.clear();
  const char* p = line.data();
  const char* e = p + line.size();
  while (p < e) {
    while (p < e && std::isspace(static_cast<unsigned char>(*p))) ++p;
    const char* b = p;
    while (p < e && !std::isspace(static_cast<unsigned char>(*p))) ++p;
    if (p > b) out.emplace_back(b, static_cast<size_t>(p - b));
  }
}

double to_value(std::string_view tok, const char* what) {  // io.hpp:42-53 (strtod rules, whole token)
  const std::string t(tok);
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(t.c_str(), &end);
  // std::stod: no conversion or ERANGE (overflow and underflow) throw
  if (t.empty() || end != t.c_str() + t.size() || end == t.c_str() || errno == ERANGE)
    fail(PMMF_DATA, std::string(what) + ": bad number '" + t + "'");
  return v;
}

int64_t to_index(std::string_view tok, const char* what) {  // io.hpp:55-61 (from_chars, whole token)
  int64_t v = 0;
  auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (r.ec != std::errc{} || r.ptr != tok.data() + tok.size())
    fail(PMMF_DATA, std::string(what) + ": bad integer '" + std::string(tok) + "'");
  return v;
}

struct Trip {
  int64_t r, c;
  double v;
};

pmmf_b200_triplets* to_c(int64_t rows, int64_t cols, const std::vector<Trip>& t, const std::vector<int64_t>* ids) {
  auto* o = static_cast<pmmf_b200_triplets*>(std::calloc(1, sizeof(pmmf_b200_triplets)));
  if (!o) fail(PMMF_INTERNAL, "host allocation failed");
  o->rows = rows;
  o->cols = cols;
  o->nnz = static_cast<int64_t>(t.size());
  const size_t n = std::max<size_t>(t.size(), 1);
  o->row = static_cast<int64_t*>(std::malloc(n * sizeof(int64_t)));
  o->col = static_cast<int64_t*>(std::malloc(n * sizeof(int64_t)));
  o->val = static_cast<double*>(std::malloc(n * sizeof(double)));
  if (!o->row || !o->col || !o->val) {
    pmmf_b200_triplets_free(o);
    fail(PMMF_INTERNAL, "host allocation failed");
  }
  for (size_t i = 0; i < t.size(); ++i) {
    o->row[i] = t[i].r;
    o->col[i] = t[i].c;
    o->val[i] = t[i].v;
  }
  if (ids) {
    o->n_ids = static_cast<int64_t>(ids->size());
    o->original_ids = static_cast<int64_t*>(std::malloc(std::max<size_t>(ids->size(), 1) * sizeof(int64_t)));
    if (!o->original_ids) {
      pmmf_b200_triplets_free(o);
      fail(PMMF_INTERNAL, "host allocation failed");
    }
    std::copy(ids->begin(), ids->end(), o->original_ids);
  }
  return o;
}

pmmf_b200_triplets* read_mm(const std::string& path) {  // io.hpp:68-129
  std::ifstream in(path);
  if (!in) fail(PMMF_DATA, "cannot open '" + path + "'");
  std::string line;
  if (!std::getline(in, line)) fail(PMMF_DATA, "matrix market: empty file");
  std::string tag, object, format, field, symmetry;
  {
    std::istringstream hdr(line);
    hdr >> tag >> object >> format >> field >> symmetry;
  }
  if (tag != "%%MatrixMarket" || lowered(object) != "matrix") fail(PMMF_DATA, "matrix market: malformed header");
  format = lowered(format);
  field = lowered(field);
  symmetry = lowered(symmetry);
  if (format != "coordinate") fail(PMMF_DATA, "matrix market: only coordinate format supported");
  if (field != "real" && field != "integer" && field != "pattern")
    fail(PMMF_DATA, "matrix market: unsupported field '" + field + "'");
  if (symmetry != "general" && symmetry != "symmetric")
    fail(PMMF_DATA, "matrix market: unsupported symmetry '" + symmetry + "'");
  const bool pattern = field == "pattern", mirror = symmetry == "symmetric";
  while (std::getline(in, line))  // comments and blank lines before the size line
    if (!line.empty() && line[0] != '%') break;
  int64_t rows = 0, cols = 0, nnz = 0;
  {
    std::istringstream dims(line);
    if (!(dims >> rows >> cols >> nnz) || rows < 0 || cols < 0 || nnz < 0)
      fail(PMMF_DATA, "matrix market: malformed size line");
  }
  std::vector<Trip> t;
  t.reserve(static_cast<size_t>(std::min<int64_t>(nnz, int64_t{1} << 28)) * (mirror ? 2 : 1));
  std::vector<std::string_view> tok;
  for (int64_t seen = 0; seen < nnz;) {
    if (!std::getline(in, line)) fail(PMMF_DATA, "matrix market: unexpected end of file");
    if (line.empty() || line[0] == '%') continue;
    split(line, tok);
    if (tok.size() < 2) fail(PMMF_DATA, "matrix market: malformed entry line");
    const int64_t i = to_index(tok[0], "matrix market") - 1;
    const int64_t j = to_index(tok[1], "matrix market") - 1;
    double v = 1.0;
    if (!pattern) {
      if (tok.size() < 3) fail(PMMF_DATA, "matrix market: missing value");
      v = to_value(tok[2], "matrix market");
    }
    if (i < 0 || i >= rows || j < 0 || j >= cols) fail(PMMF_DATA, "matrix market: index out of range");
    if (!std::isfinite(v)) fail(PMMF_DATA, "matrix market: non-finite value");
    t.push_back({i, j, v});
    if (mirror && i != j) t.push_back({j, i, v});
    ++seen;
  }
  return to_c(rows, cols, t, nullptr);
}

pmmf_b200_triplets* read_edges(const std::string& path) {  // io.hpp:158-208
  std::ifstream in(path);
  if (!in) fail(PMMF_DATA, "cannot open '" + path + "'");
  std::string line;
  std::vector<Trip> raw;
  std::vector<std::string_view> tok;
  bool any = false;
  while (std::getline(in, line)) {
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    split(line, tok);
    if (tok.empty()) continue;
    if (tok.size() < 2) fail(PMMF_DATA, "edge list: line with a single token");
    any = true;
    const int64_t u = to_index(tok[0], "edge list");
    const int64_t v = to_index(tok[1], "edge list");
    double w = 1.0;
    if (tok.size() >= 3) w = to_value(tok[2], "edge list");
    if (!std::isfinite(w)) fail(PMMF_DATA, "edge list: non-finite weight");
    raw.push_back({u, v, w});
  }
  if (!any) fail(PMMF_DATA, "edge list: no edges found");
  std::vector<int64_t> ids;
  ids.reserve(raw.size() * 2);
  for (const Trip& e : raw) {
    ids.push_back(e.r);
    ids.push_back(e.c);
  }
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  auto id_of = [&](int64_t x) { return static_cast<int64_t>(std::lower_bound(ids.begin(), ids.end(), x) - ids.begin()); };
  std::vector<Trip> t;
  t.reserve(raw.size() * 2);
  for (const Trip& e : raw) {
    const int64_t u = id_of(e.r), v = id_of(e.c);
    t.push_back({u, v, e.v});
    if (u != v) t.push_back({v, u, e.v});
  }
  const int64_t n = static_cast<int64_t>(ids.size());
  return to_c(n, n, t, &ids);
}

void write_mm(const std::string& path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* r, const int64_t* c,
              const double* v) {  // io.hpp:131-147
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(PMMF_DATA, "cannot open '" + path + "' for writing");
  std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", static_cast<long long>(rows),
               static_cast<long long>(cols), static_cast<long long>(nnz));
  for (int64_t i = 0; i < nnz; ++i)
    std::fprintf(f, "%lld %lld %.17g\n", static_cast<long long>(r[i] + 1), static_cast<long long>(c[i] + 1), v[i]);
  const bool ok = std::fclose(f) == 0;
  if (!ok) fail(PMMF_DATA, "cannot write '" + path + "'");
}

// ------------------------------------------------------------ device
// first offending triplet: range before sign for the same triplet, as the
// reference's single loop checks them (io.hpp:215-219)
__global__ void k_lap_check(int64_t nnz, int64_t n, const int64_t* __restrict__ r, const int64_t* __restrict__ c,
                            const double* __restrict__ v, unsigned long long* __restrict__ first) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= nnz) return;
  int code = 0;
  if (r[t] < 0 || r[t] >= n || c[t] < 0 || c[t] >= n) code = 1;
  else if (v[t] < 0.0) code = 2;
  if (code) atomicMin(first, (static_cast<unsigned long long>(t) << 2) | static_cast<unsigned long long>(code));
}

__global__ void k_lap_keys(int64_t nnz, const int64_t* __restrict__ r, uint32_t* __restrict__ key,
                           uint32_t* __restrict__ pos, int32_t* __restrict__ cnt) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= nnz) return;
  key[t] = static_cast<uint32_t>(r[t]);
  pos[t] = static_cast<uint32_t>(t);
  atomicAdd(cnt + r[t], 1);
}

// degree of row i: 0.0 + its weights in input order (io.hpp:219)
__global__ void k_lap_degree(int64_t n, const int64_t* __restrict__ ptr, const uint32_t* __restrict__ pos,
                             const double* __restrict__ v, double shift, int64_t nnz, int64_t* __restrict__ orow,
                             int64_t* __restrict__ ocol, double* __restrict__ oval) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (int64_t x = ptr[i]; x < ptr[i + 1]; ++x) d = dadd(d, v[pos[x]]);
  orow[nnz + i] = i;
  ocol[nnz + i] = i;
  oval[nnz + i] = dadd(d, shift);
}

__global__ void k_lap_offdiag(int64_t nnz, const int64_t* __restrict__ r, const int64_t* __restrict__ c,
                              const double* __restrict__ v, int64_t* __restrict__ orow, int64_t* __restrict__ ocol,
                              double* __restrict__ oval) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= nnz) return;
  orow[t] = r[t];
  ocol[t] = c[t];
  oval[t] = -v[t];
}

__global__ void k_widen32(int64_t n, const int32_t* __restrict__ a, int64_t* __restrict__ b) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) b[i] = a[i];
  if (i == n) b[i] = 0;
}

// unordered pair key (min, max), both offset into [0, 2^32)
__global__ void k_sym_keys(int64_t nnz, const int64_t* __restrict__ r, const int64_t* __restrict__ c,
                           uint64_t* __restrict__ key, uint32_t* __restrict__ pos, int* __restrict__ bad) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= nnz) return;
  const int64_t i = min(r[t], c[t]), j = max(r[t], c[t]);
  if (i < INT_MIN || j > INT_MAX) atomicExch(bad, 1);
  key[t] = (static_cast<uint64_t>(i + 2147483648LL) << 32) | static_cast<uint64_t>(j + 2147483648LL);
  pos[t] = static_cast<uint32_t>(t);
}

__global__ void k_sym_heads(int64_t nnz, const uint64_t* __restrict__ key, int64_t* __restrict__ head) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= nnz) return;
  head[t] = (t == 0 || key[t] != key[t - 1]) ? 1 : 0;
}

__global__ void k_sym_starts(int64_t nnz, const int64_t* __restrict__ head, const int64_t* __restrict__ hpos,
                             int64_t* __restrict__ start, int64_t* __restrict__ width, const uint64_t* __restrict__ key) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= nnz || !head[t]) return;
  const int64_t g = hpos[t];
  start[g] = t;
  width[g] = (key[t] >> 32) == (key[t] & 0xffffffffu) ? 1 : 2;
}

// group g: sum from 0.0 in input order (std::map accumulator, io.hpp:233-237)
__global__ void k_sym_emit(int64_t G, int64_t nnz, const int64_t* __restrict__ start, const int64_t* __restrict__ opos,
                           const uint64_t* __restrict__ key, const uint32_t* __restrict__ pos,
                           const double* __restrict__ v, int64_t* __restrict__ orow, int64_t* __restrict__ ocol,
                           double* __restrict__ oval) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= G) return;
  const int64_t b = start[g], e = g + 1 < G ? start[g + 1] : nnz;
  double s = 0.0;
  for (int64_t x = b; x < e; ++x) s = dadd(s, v[pos[x]]);
  const int64_t i = static_cast<int64_t>(key[b] >> 32) - 2147483648LL;
  const int64_t j = static_cast<int64_t>(key[b] & 0xffffffffu) - 2147483648LL;
  const int64_t o = opos[g];
  if (i == j) {
    orow[o] = i;
    ocol[o] = i;
    oval[o] = dmul(2.0, s);
  } else {
    orow[o] = i;
    ocol[o] = j;
    oval[o] = s;
    orow[o + 1] = j;
    ocol[o + 1] = i;
    oval[o + 1] = s;
  }
}

template <typename T>
void scan_excl(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
  PMMF_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, n, s));
}

// inputs on the device (uploaded when given on the host)
struct In3 {
  DBuf<int64_t> r, c;
  DBuf<double> v;
  const int64_t* pr = nullptr;
  const int64_t* pc = nullptr;
  const double* pv = nullptr;
  In3(int64_t nnz, const int64_t* r0, const int64_t* c0, const double* v0, bool on_dev, cudaStream_t s) {
    if (on_dev) {
      pr = r0;
      pc = c0;
      pv = v0;
      return;
    }
    r.alloc(std::max<int64_t>(nnz, 1), s);
    c.alloc(std::max<int64_t>(nnz, 1), s);
    v.alloc(std::max<int64_t>(nnz, 1), s);
    r.upload(r0, nnz);
    c.upload(c0, nnz);
    v.upload(v0, nnz);
    pr = r.get();
    pc = c.get();
    pv = v.get();
  }
};

struct Out3 {
  DBuf<int64_t> r, c;
  DBuf<double> v;
  int64_t* pr;
  int64_t* pc;
  double* pv;
  Out3(int64_t cap, int64_t* r0, int64_t* c0, double* v0, bool on_dev, cudaStream_t s) {
    if (on_dev) {
      pr = r0;
      pc = c0;
      pv = v0;
      return;
    }
    r.alloc(std::max<int64_t>(cap, 1), s);
    c.alloc(std::max<int64_t>(cap, 1), s);
    v.alloc(std::max<int64_t>(cap, 1), s);
    pr = r.get();
    pc = c.get();
    pv = v.get();
  }
  void download(int64_t n, int64_t* r0, int64_t* c0, double* v0, bool on_dev, cudaStream_t s) {
    if (on_dev || n == 0) return;
    r.download(r0, n);
    c.download(c0, n);
    v.download(v0, n);
    PMMF_CUDA(cudaStreamSynchronize(s));
  }
};

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { PMMF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
};

void laplacian_dev(int64_t n, int64_t nnz, const int64_t* r0, const int64_t* c0, const double* v0, double shift,
                   bool on_dev, int64_t* orow, int64_t* ocol, double* oval) {  // io.hpp:212-228
  if (n < 0 || nnz < 0) fail(PMMF_INVALID_ARGUMENT, "laplacian: negative size");
  if (n >= (int64_t{1} << 32) || nnz >= (int64_t{1} << 32))
    fail(PMMF_INVALID_ARGUMENT, "laplacian: more than 2^32 rows or entries");
  Stream st;
  cudaStream_t s = st.s;
  In3 in(nnz, r0, c0, v0, on_dev, s);
  Out3 out(nnz + n, orow, ocol, oval, on_dev, s);
  if (nnz > 0) {
    DBuf<unsigned long long> first(1, s);
    first.fill_bytes(0xff);
    PMMF_LAUNCH(k_lap_check, blocks_for(nnz, kThreads), kThreads, 0, s, nnz, n, in.pr, in.pc, in.pv, first.get());
    const unsigned long long f = first.to_host(1)[0];
    if (f != ~0ull) fail(PMMF_DATA, (f & 3) == 1 ? "laplacian: index out of range" : "laplacian: negative weight");
  }
  DBuf<int32_t> cnt(n + 1, s);
  cnt.zero();
  DBuf<uint32_t> k1(std::max<int64_t>(nnz, 1), s), k2(std::max<int64_t>(nnz, 1), s), p1(std::max<int64_t>(nnz, 1), s),
      p2(std::max<int64_t>(nnz, 1), s);
  DBuf<int64_t> c64(n + 1, s), ptr(n + 1, s);
  if (nnz > 0) {
    PMMF_LAUNCH(k_lap_keys, blocks_for(nnz, kThreads), kThreads, 0, s, nnz, in.pr, k1.get(), p1.get(), cnt.get());
    int bits = 1;
    while (bits < 32 && (int64_t{1} << bits) < n) ++bits;
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k1.get(), k2.get(), p1.get(), p2.get(), nnz, 0, bits, s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, k1.get(), k2.get(), p1.get(), p2.get(), nnz, 0, bits, s));
  }
  PMMF_LAUNCH(k_widen32, blocks_for(n + 1, kThreads), kThreads, 0, s, n, cnt.get(), c64.get());
  scan_excl(c64.get(), ptr.get(), n + 1, s);
  PMMF_LAUNCH(k_lap_offdiag, blocks_for(nnz, kThreads), kThreads, 0, s, nnz, in.pr, in.pc, in.pv, out.pr, out.pc,
              out.pv);
  PMMF_LAUNCH(k_lap_degree, blocks_for(n, kThreads), kThreads, 0, s, n, ptr.get(), p2.get(), in.pv, shift, nnz,
              out.pr, out.pc, out.pv);
  out.download(nnz + n, orow, ocol, oval, on_dev, s);
  PMMF_CUDA(cudaStreamSynchronize(s));
}

int64_t symmetrize_dev(int64_t nnz, const int64_t* r0, const int64_t* c0, const double* v0, bool on_dev,
                       int64_t* orow, int64_t* ocol, double* oval) {  // io.hpp:231-250
  if (nnz < 0) fail(PMMF_INVALID_ARGUMENT, "symmetrize: negative size");
  if (nnz >= (int64_t{1} << 32)) fail(PMMF_INVALID_ARGUMENT, "symmetrize: more than 2^32 entries");
  if (nnz == 0) return 0;
  Stream st;
  cudaStream_t s = st.s;
  In3 in(nnz, r0, c0, v0, on_dev, s);
  DBuf<uint64_t> k1(nnz, s), k2(nnz, s);
  DBuf<uint32_t> p1(nnz, s), p2(nnz, s);
  DBuf<int> bad(1, s);
  bad.zero();
  PMMF_LAUNCH(k_sym_keys, blocks_for(nnz, kThreads), kThreads, 0, s, nnz, in.pr, in.pc, k1.get(), p1.get(), bad.get());
  if (bad.to_host(1)[0]) fail(PMMF_OUT_OF_RANGE, "symmetrize: index outside the 32-bit range");
  {
    size_t tmp = 0;
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k1.get(), k2.get(), p1.get(), p2.get(), nnz, 0, 64, s));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1, s);
    PMMF_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, k1.get(), k2.get(), p1.get(), p2.get(), nnz, 0, 64, s));
  }
  DBuf<int64_t> head(nnz + 1, s), hpos(nnz + 1, s);
  head.zero();
  PMMF_LAUNCH(k_sym_heads, blocks_for(nnz, kThreads), kThreads, 0, s, nnz, k2.get(), head.get());
  scan_excl(head.get(), hpos.get(), nnz + 1, s);
  const int64_t G = hpos.to_host(nnz + 1)[nnz];
  DBuf<int64_t> start(G, s), width(G + 1, s), opos(G + 1, s);
  width.zero();
  PMMF_LAUNCH(k_sym_starts, blocks_for(nnz, kThreads), kThreads, 0, s, nnz, head.get(), hpos.get(), start.get(),
              width.get(), k2.get());
  scan_excl(width.get(), opos.get(), G + 1, s);
  const int64_t total = opos.to_host(G + 1)[G];
  Out3 out(total, orow, ocol, oval, on_dev, s);
  PMMF_LAUNCH(k_sym_emit, blocks_for(G, kThreads), kThreads, 0, s, G, nnz, start.get(), opos.get(), k2.get(), p2.get(),
              in.pv, out.pr, out.pc, out.pv);
  out.download(total, orow, ocol, oval, on_dev, s);
  PMMF_CUDA(cudaStreamSynchronize(s));
  return total;
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  return guarded_call(err, errlen, [](void* c) { (*static_cast<F*>(c))(); }, &f);
}

}  // namespace
}  // namespace pmmf_b200

using namespace pmmf_b200;

extern "C" {

void pmmf_b200_triplets_free(pmmf_b200_triplets* t) {
  if (!t) return;
  std::free(t->row);
  std::free(t->col);
  std::free(t->val);
  std::free(t->original_ids);
  std::free(t);
}

int pmmf_b200_read_matrix_market(const char* path, pmmf_b200_triplets** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!path || !out) fail(PMMF_INVALID_ARGUMENT, "read_matrix_market: null argument");
    *out = read_mm(path);
  });
}

int pmmf_b200_read_edge_list(const char* path, pmmf_b200_triplets** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!path || !out) fail(PMMF_INVALID_ARGUMENT, "read_edge_list: null argument");
    *out = read_edges(path);
  });
}

int pmmf_b200_write_matrix_market(const char* path, int64_t rows, int64_t cols, int64_t nnz, const int64_t* r,
                                  const int64_t* c, const double* v, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!path || (nnz > 0 && (!r || !c || !v))) fail(PMMF_INVALID_ARGUMENT, "write_matrix_market: null argument");
    write_mm(path, rows, cols, nnz, r, c, v);
  });
}

int pmmf_b200_laplacian(int64_t n, int64_t nnz, const int64_t* r, const int64_t* c, const double* v, double shift,
                        int32_t on_device, int32_t device, int64_t* out_r, int64_t* out_c, double* out_v, char* err,
                        size_t errlen) {
  return guarded(err, errlen, [&] {
    if ((nnz > 0 && (!r || !c || !v)) || (nnz + n > 0 && (!out_r || !out_c || !out_v)))
      fail(PMMF_INVALID_ARGUMENT, "laplacian: null argument");
    PMMF_CUDA(cudaSetDevice(device));
    laplacian_dev(n, nnz, r, c, v, shift, on_device != 0, out_r, out_c, out_v);
  });
}

int pmmf_b200_symmetrize(int64_t nnz, const int64_t* r, const int64_t* c, const double* v, int32_t on_device,
                         int32_t device, int64_t* out_nnz, int64_t* out_r, int64_t* out_c, double* out_v, char* err,
                         size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!out_nnz || (nnz > 0 && (!r || !c || !v || !out_r || !out_c || !out_v)))
      fail(PMMF_INVALID_ARGUMENT, "symmetrize: null argument");
    PMMF_CUDA(cudaSetDevice(device));
    *out_nnz = symmetrize_dev(nnz, r, c, v, on_device != 0, out_r, out_c, out_v);
  });
}

}  // extern "C"
