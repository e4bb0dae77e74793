// setup.cu -- problem setup (matio.py:104-275): Matrix
// Market ingest on the host in native code, operator-norm power iterations on
// the device, so paper-protocol and c5-scale setup is not host-bound.
//
// sscg_mm_parse follows read_matrix_market (matio.py:104-184) token for token:
// header checks, comment / blank skipping, `i j value` entries with Python's
// int()/float() acceptance for plain decimal text, the same error messages and
// line numbers; a symmetric file appends the mirrored off-diagonal entries
// after the stored ones; from_coo (matio.py:87-101) is then a stable row
// bucket, a per-row sort by column and duplicate summation in that order (the
// reference sums pairs identically; with three or more copies of one entry its
// unstable sort may add them in another order).
//
// sscg_power_iteration is _power_iteration (matio.py:229-244) with the matvec
// A v, |A| v or shift*v - A v (csr_matvec rounding) on the device; norms and
// dots are fixed-order tree sums, so estimates agree with the reference to the
// power method's tolerance, not bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"
#include "rowops.cuh"

struct sscg_mm {
  int64_t n = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col;
  std::vector<double> val;
};

namespace {
thread_local int g_mm_line = 0;

int mm_fail(int line, const char* fmt, ...) {
  char buf[400];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_mm_line = line;
  if (line > 0) {
    char full[480];
    snprintf(full, sizeof(full), "%s (line %d)", buf, line);
    return sscg_fail(SSCG_EFORMAT, "%s", full);
  }
  return sscg_fail(SSCG_EFORMAT, "%s", buf);
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

// str.split() of one line
void split(const char* b, const char* e, std::vector<std::string>& out) {
  out.clear();
  while (b < e) {
    while (b < e && is_space(*b)) ++b;
    const char* s = b;
    while (b < e && !is_space(*b)) ++b;
    if (b > s) out.emplace_back(s, b);
  }
}

std::string lower(std::string s) {
  for (char& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

// Python int() of a plain decimal token
bool py_int(const std::string& t, int64_t* v) {
  const char* s = t.c_str();
  if (*s == '+' || *s == '-') ++s;
  if (!*s) return false;
  for (const char* q = s; *q; ++q)
    if (*q < '0' || *q > '9') return false;
  errno = 0;
  char* end = nullptr;
  const long long x = strtoll(t.c_str(), &end, 10);
  if (errno || *end) return false;
  *v = x;
  return true;
}

// Python float() of a decimal / inf / nan token (no hex floats)
bool py_float(const std::string& t, double* v) {
  if (t.empty()) return false;
  for (char c : t)
    if (c == 'x' || c == 'X' || c == 'p' || c == 'P') return false;
  char* end = nullptr;
  const double x = strtod(t.c_str(), &end);
  if (*end || end == t.c_str()) return false;
  *v = x;
  return true;
}

bool line_blank(const char* b, const char* e) {
  for (; b < e; ++b)
    if (!is_space(*b)) return false;
  return true;
}
}  // namespace

extern "C" {

int sscg_mm_error_line(void) { return g_mm_line; }

int sscg_mm_parse(const char* text, int64_t len, sscg_mm** out, int64_t* n_out, int64_t* nnz_out,
                  int32_t* symmetric_out) {
  g_mm_line = 0;
  if (!text || !out || !n_out || !nnz_out) return sscg_fail(SSCG_EINVAL, "NULL argument");
  *out = nullptr;
  const char* p = text;
  const char* end = text + len;
  auto next_line = [&](const char** b, const char** e) -> bool {
    if (p >= end) return false;
    *b = p;
    const char* q = (const char*)memchr(p, '\n', (size_t)(end - p));
    *e = q ? q : end;
    p = q ? q + 1 : end;
    return true;
  };
  const char *lb, *le;
  std::vector<std::string> tok;
  if (!next_line(&lb, &le) || strncmp(lb, "%%MatrixMarket", 14) != 0 || le - lb < 14)
    return mm_fail(1, "missing %%%%MatrixMarket header");
  split(lb, le, tok);
  if (tok.size() != 5) return mm_fail(1, "malformed header");
  const std::string obj = lower(tok[1]), fmt = lower(tok[2]), fld = lower(tok[3]),
                    sym = lower(tok[4]);
  if (obj != "matrix" || fmt != "coordinate")
    return mm_fail(1, "unsupported object/format '%s %s'", obj.c_str(), fmt.c_str());
  if (fld == "complex") return mm_fail(1, "complex field not supported");
  if (fld == "pattern") return mm_fail(1, "pattern-only files carry no values");
  if (fld != "real" && fld != "integer") return mm_fail(1, "unsupported field '%s'", fld.c_str());
  if (sym != "general" && sym != "symmetric")
    return mm_fail(1, "unsupported symmetry '%s'", sym.c_str());
  int line_no = 1;
  bool have_size = false;
  while (next_line(&lb, &le)) {
    ++line_no;
    if ((le > lb && *lb == '%') || line_blank(lb, le)) continue;
    have_size = true;
    break;
  }
  if (!have_size) return mm_fail(line_no, "missing size line");
  split(lb, le, tok);
  int64_t m = 0, n = 0, nnz = 0;
  if (tok.size() != 3 || !py_int(tok[0], &m) || !py_int(tok[1], &n) || !py_int(tok[2], &nnz))
    return mm_fail(line_no, "size line must be 'rows cols nnz'");
  if (m != n) return mm_fail(line_no, "matrix must be square, got %lldx%lld", (long long)m, (long long)n);
  if (n < 0 || nnz < 0) return mm_fail(line_no, "size line must be 'rows cols nnz'");
  if (n >= ((int64_t)1 << 31)) return mm_fail(line_no, "n exceeds int32 column indices");
  std::vector<int64_t> ri, ci;
  std::vector<double> vv;
  ri.reserve((size_t)nnz);
  ci.reserve((size_t)nnz);
  vv.reserve((size_t)nnz);
  int64_t k = 0;
  while (next_line(&lb, &le)) {
    ++line_no;
    if (line_blank(lb, le) || (le > lb && *lb == '%')) continue;
    split(lb, le, tok);
    if (tok.size() != 3) return mm_fail(line_no, "entry line must be 'i j value'");
    int64_t i = 0, j = 0;
    double v = 0.0;
    if (!py_int(tok[0], &i) || !py_int(tok[1], &j) || !py_float(tok[2], &v))
      return mm_fail(line_no, "could not parse entry");
    --i;
    --j;
    if (k >= nnz) return mm_fail(line_no, "more entries than declared");
    if (!(0 <= i && i < n && 0 <= j && j < n)) return mm_fail(line_no, "index out of range");
    ri.push_back(i);
    ci.push_back(j);
    vv.push_back(v);
    ++k;
  }
  if (k != nnz)
    return mm_fail(line_no, "expected %lld entries, found %lld", (long long)nnz, (long long)k);
  if (sym == "symmetric") {  // matio.py:174-180: mirrored strict triangle appended
    const int64_t k0 = k;
    for (int64_t e = 0; e < k0; ++e)
      if (ri[e] != ci[e]) {
        ri.push_back(ci[e]);
        ci.push_back(ri[e]);
        vv.push_back(vv[e]);
      }
  }
  // from_coo: stable row buckets, per-row column sort, duplicates summed
  auto* mm = new sscg_mm();
  mm->n = n;
  const int64_t total = (int64_t)ri.size();
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t e = 0; e < total; ++e) ++cnt[ri[e] + 1];
  for (int64_t r = 0; r < n; ++r) cnt[r + 1] += cnt[r];
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1), order((size_t)total);
  for (int64_t e = 0; e < total; ++e) order[pos[ri[e]]++] = e;
  mm->row_ptr.assign(n + 1, 0);
  for (int64_t r = 0; r < n; ++r) {
    auto b = order.begin() + cnt[r], e = order.begin() + cnt[r + 1];
    std::stable_sort(b, e, [&](int64_t x, int64_t y) { return ci[x] < ci[y]; });
    for (auto it = b; it != e;) {
      const int64_t c = ci[*it];
      double s = vv[*it];
      for (++it; it != e && ci[*it] == c; ++it) s += vv[*it];
      mm->col.push_back((int32_t)c);
      mm->val.push_back(s);
    }
    mm->row_ptr[r + 1] = (int64_t)mm->col.size();
  }
  if (sym == "general") {  // pattern_is_symmetric over stored nonzeros (matio.py:64-67)
    auto has_nz = [&](int64_t r, int64_t c) {
      const auto b = mm->col.begin() + mm->row_ptr[r], e = mm->col.begin() + mm->row_ptr[r + 1];
      const auto it = std::lower_bound(b, e, (int32_t)c);
      return it != e && *it == (int32_t)c && mm->val[it - mm->col.begin()] != 0.0;
    };
    for (int64_t r = 0; r < n; ++r)
      for (int64_t e = mm->row_ptr[r]; e < mm->row_ptr[r + 1]; ++e)
        if (mm->val[e] != 0.0 && !has_nz(mm->col[e], r)) {
          delete mm;
          return mm_fail(0, "general file without structurally symmetric pattern");
        }
  }
  *out = mm;
  *n_out = n;
  *nnz_out = (int64_t)mm->col.size();
  if (symmetric_out) *symmetric_out = sym == "symmetric";
  return SSCG_OK;
}

int sscg_mm_take(sscg_mm* mm, int64_t* row_ptr, int32_t* col_idx, double* values) {
  if (!mm || !row_ptr || (!mm->col.empty() && (!col_idx || !values)))
    return sscg_fail(SSCG_EINVAL, "NULL argument");
  std::copy(mm->row_ptr.begin(), mm->row_ptr.end(), row_ptr);
  std::copy(mm->col.begin(), mm->col.end(), col_idx);
  std::copy(mm->val.begin(), mm->val.end(), values);
  return SSCG_OK;
}

void sscg_mm_free(sscg_mm* mm) { delete mm; }

}  // extern "C"

// ---------------------------------------------------------------------------
// power iteration kernels (CSR rows, csr_matvec order)
namespace {
constexpr int PW_T = ROWS_PER_CTA;

__device__ __forceinline__ double pw_row(const Ctx& c, int mode, double shift, int64_t i,
                                         const double* v) {
  const int beg = c.rp[i], end = c.rp[i + 1];
  double acc = 0.0;
  for (int j = beg; j < end; ++j) {
    const double a = __ldg(c.val + j);
    acc = __dadd_rn(acc, __dmul_rn(mode == 1 ? fabs(a) : a, __ldg(v + c.col[j])));
  }
  return mode == 2 ? __dsub_rn(__dmul_rn(shift, v[i]), acc) : acc;  // norm_a*v - spmv(a, v)
}

__device__ __forceinline__ bool pw_last(int* counter) {
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// out = op(v); *res = dot(dotv ? dotv : out, out) (fixed-order sum)
__global__ void __launch_bounds__(PW_T) k_pw_apply(Ctx c, int mode, double shift, const double* v,
                                                   double* out, const double* dotv, double* res) {
  __shared__ double sm[PW_T / 32];
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * PW_T;
  for (int64_t i = (int64_t)blockIdx.x * PW_T + threadIdx.x; i < c.n; i += stride) {
    const double w = pw_row(c, mode, shift, i, v);
    out[i] = w;
    s = fma(dotv ? dotv[i] : w, w, s);
  }
  s = block_sum<PW_T>(s, sm);
  if (threadIdx.x == 0) c.part_t[blockIdx.x] = s;
  if (!pw_last(&c.st->gram_count)) return;
  double t = 0.0;
  for (int j = threadIdx.x; j < (int)gridDim.x; j += PW_T) t += c.part_t[j];
  t = block_sum<PW_T>(t, sm);
  if (threadIdx.x == 0) {
    *res = t;
    c.st->gram_count = 0;
  }
}

__global__ void k_pw_scale(int64_t n, const double* w, double inv_norm_div, double* v) {
  // v = w / nw (numpy true division, element by element)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __ddiv_rn(w[i], inv_norm_div);
}
}  // namespace

// host side lives with the plan (plan.cu): these launchers are its interface
void launch_pw_apply(const Ctx& c, int mode, double shift, const double* v, double* out,
                     const double* dotv, double* res, cudaStream_t s) {
  k_pw_apply<<<c.red_n, PW_T, 0, s>>>(c, mode, shift, v, out, dotv, res);
}
void launch_pw_scale(int64_t n, const double* w, double nw, double* v, cudaStream_t s) {
  k_pw_scale<<<(int)std::min<int64_t>((n + 255) / 256, 4 * NUM_SMS), 256, 0, s>>>(n, w, nw, v);
}
