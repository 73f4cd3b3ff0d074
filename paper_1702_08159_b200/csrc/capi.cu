// extern "C" boundary of libmckernel_b200.so (declared in include/mckernel_b200.h).
// Argument validation mirrors the reference's ValueError checks; messages keep
// the reference's wording where a reference test matches on it
// (wht.py:36-38,136-137,155-158; fastfood.py:37-53,170-172,182-183).
#include <cstdarg>
#include <cmath>
#include <string>

#include "mck_common.cuh"
#include "tables.cuh"

namespace mck {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int fail_value(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return MCK_ERR_VALUE;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return MCK_OK;
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return MCK_ERR_CUDA;
}

int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

// implemented in the kernel translation units
int stream_hashes(uint64_t, uint64_t, int64_t, uint64_t*, cudaStream_t);
int stream_uniforms(uint64_t, uint64_t, int64_t, double*, cudaStream_t);
int stream_signs(uint64_t, uint64_t, int64_t, double*, cudaStream_t);
int stream_gaussian_pairs(uint64_t, uint64_t, int64_t, double*, cudaStream_t);
int fisher_yates(uint64_t, uint64_t, uint64_t, int32_t, int64_t, int32_t*, cudaStream_t);
int build_factors(const TablesView&, uint64_t, int32_t, int32_t, cudaStream_t);
int prepare_tables(const TablesView&, float, int, cudaStream_t, bool);
template <class V> int fwht_fast(V*, int64_t, int64_t, cudaStream_t);
int fwht_parity(float*, int64_t, int64_t, cudaStream_t);
int fastfood_run(const TablesView&, int32_t, double, const float*, int64_t, int64_t,
                 const int32_t*, bool, bool, float*, int64_t, int, cudaStream_t);
int head_forward(const float*, int64_t, int64_t, int64_t, const double*, const double*, int32_t,
                 const int32_t*, const int32_t*, int64_t, double*, double*, double*, int64_t*, void*, cudaStream_t);
int head_backward(const float*, int64_t, int64_t, int64_t, const double*, int32_t, double*,
                  double*, void*, cudaStream_t);
int head_backward_sgd(const float*, int64_t, int64_t, int64_t, const double*, int32_t, double*,
                      double*, double, double, void*, cudaStream_t);
int head_sgd_update(double*, double*, const double*, const double*, int64_t, int32_t, double,
                    double, cudaStream_t);
int64_t head_scratch_bytes(int64_t, int64_t, int32_t);
int64_t fused_scratch_bytes(int64_t, int64_t, int32_t, int32_t, bool);
int fused_forward(const TablesView&, int32_t, double, const float*, int64_t, int64_t,
                  const int32_t*, const float*, const double*, int32_t, const int32_t*,
                  const int32_t*, int64_t, double*, double*, double*, double*, int64_t*, void*,
                  int32_t, cudaStream_t);
int fused_backward(const TablesView&, int32_t, double, const float*, int64_t, int64_t,
                   const int32_t*, const double*, int32_t, float*, double*, float*, double*,
                   double, double, void*, int32_t, cudaStream_t);
int fused_backward_range(const TablesView&, int32_t, double, const float*, int64_t, int64_t,
                         const int32_t*, const double*, int32_t, int32_t, int32_t, float*, int64_t,
                         int64_t, int64_t, float*, double, double, void*, int32_t, cudaStream_t);
int fused_bias_grad(const double*, int64_t, int32_t, double*, cudaStream_t);
int fused_apply_bucket(float*, int64_t, int32_t, int32_t, int32_t, int32_t, const float*, double, double,
                       double*, const double*, cudaStream_t);

static bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
static int64_t next_pow2(int64_t d) {
  int64_t n = 1;
  while (n < d) n <<= 1;
  return n;
}
static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static void tables_scale(int64_t n, double sigma, float* scale, int* fold) {
  const float s = (float)(1.0 / (sigma * std::sqrt((double)n)));
  int ex = 0;
  *scale = s;
  *fold = std::frexp(s, &ex) == 0.5f ? 1 : 0;
}

static int check_spec(int64_t input_dim, int32_t E, double sigma) {
  if (input_dim < 1) return fail_value("input_dim must be positive");
  if (E < 1) return fail_value("expansions must be positive");
  if (!(sigma > 0.0)) return fail_value("sigma must be positive");
  if (next_pow2(input_dim) > (int64_t(1) << 20))
    return fail_value("padded_dim %lld exceeds the supported maximum 2^20",
                      (long long)next_pow2(input_dim));
  return MCK_OK;
}

}  // namespace mck

using namespace mck;

extern "C" {

int mck_abi_version(void) { return 1; }

const char* mck_last_error(void) { return g_last_error.c_str(); }

uint64_t mck_stream_key(uint64_t seed, const char* label, uint64_t block) {
  return stream_key(seed, label ? label : "", block);
}

int mck_stream_hashes(uint64_t key, uint64_t c0, int64_t count, uint64_t* out, void* st) {
  if (count < 0) return fail_value("count must be non-negative");
  return stream_hashes(key, c0, count, out, S(st));
}
int mck_stream_uniforms(uint64_t key, uint64_t c0, int64_t count, double* out, void* st) {
  if (count < 0) return fail_value("count must be non-negative");
  return stream_uniforms(key, c0, count, out, S(st));
}
int mck_stream_signs(uint64_t key, uint64_t c0, int64_t count, double* out, void* st) {
  if (count < 0) return fail_value("count must be non-negative");
  return stream_signs(key, c0, count, out, S(st));
}
int mck_stream_gaussian_pairs(uint64_t key, uint64_t c0, int64_t pairs, double* out, void* st) {
  if (pairs < 0) return fail_value("count must be non-negative");
  return stream_gaussian_pairs(key, c0, pairs, out, S(st));
}
int mck_fisher_yates(uint64_t seed, const char* label, uint64_t block0, int32_t count, int64_t n,
                     int32_t* out, void* st) {
  if (n < 1) return fail_value("empty permutation");
  if (n > (int64_t(1) << 31) - 1) return fail_value("permutation too long");
  return fisher_yates(seed, fnv1a64(label ? label : ""), block0, count, n, out, S(st));
}

int64_t mck_tables_bytes(int64_t n, int32_t E) {
  if (n < 1 || E < 1) return 0;
  return tables_layout(n, E, nullptr, nullptr);
}

int mck_tables_build(void* tables, int64_t input_dim, int32_t E, int32_t kind, double sigma,
                     int32_t t, uint64_t seed, void* st) {
  MCK_TRY(check_spec(input_dim, E, sigma));
  if (kind != MCK_KERNEL_RBF && kind != MCK_KERNEL_MATERN) return fail_value("unknown kernel kind");
  if (kind == MCK_KERNEL_MATERN && t < 1) return fail_value("t must be a positive integer");
  if (!tables) return fail_value("tables buffer is NULL");
  const int64_t n = next_pow2(input_dim);
  if (kind == MCK_KERNEL_MATERN && n > 16384)
    return fail_value("Matern calibration supports padded_dim <= 16384 (got %lld): it costs t*n^2 "
                      "gaussians per block", (long long)n);
  TablesView tv;
  tables_layout(n, E, (char*)tables, &tv);
  MCK_TRY(build_factors(tv, seed, kind, t, S(st)));
  float scale;
  int fold;
  tables_scale(n, sigma, &scale, &fold);
  return prepare_tables(tv, scale, fold, S(st), false);
}

int mck_tables_from_factors(void* tables, int64_t input_dim, int32_t E, double sigma,
                            const float* b, const int32_t* perm, const float* g, const float* c,
                            void* st) {
  MCK_TRY(check_spec(input_dim, E, sigma));
  if (!tables || !b || !perm || !g || !c) return fail_value("NULL factor pointer");
  const int64_t n = next_pow2(input_dim);
  TablesView tv;
  tables_layout(n, E, (char*)tables, &tv);
  const size_t bytes = (size_t)n * E * 4;
  MCK_TRY(check_cuda(cudaMemcpyAsync(tv.b, b, bytes, cudaMemcpyDeviceToDevice, S(st)), "copy b"));
  MCK_TRY(check_cuda(cudaMemcpyAsync(tv.perm, perm, bytes, cudaMemcpyDeviceToDevice, S(st)), "copy perm"));
  MCK_TRY(check_cuda(cudaMemcpyAsync(tv.g, g, bytes, cudaMemcpyDeviceToDevice, S(st)), "copy g"));
  MCK_TRY(check_cuda(cudaMemcpyAsync(tv.c, c, bytes, cudaMemcpyDeviceToDevice, S(st)), "copy c"));
  float scale;
  int fold;
  tables_scale(n, sigma, &scale, &fold);
  return prepare_tables(tv, scale, fold, S(st), true);
}

int mck_tables_factors(void* tables, int64_t n, int32_t E, float** b, int32_t** perm, float** g,
                       float** c) {
  if (!is_pow2(n) || E < 1) return fail_value("bad table geometry");
  TablesView tv;
  tables_layout(n, E, (char*)tables, &tv);
  if (b) *b = tv.b;
  if (perm) *perm = tv.perm;
  if (g) *g = tv.g;
  if (c) *c = tv.c;
  return MCK_OK;
}

int mck_fwht_f32(float* data, int64_t rows, int64_t n, int32_t variant, void* st) {
  if (!is_pow2(n)) return fail_value("length %lld is not a power of two", (long long)n);
  if (rows < 0) return fail_value("rows must be non-negative");
  if (n > (int64_t(1) << 20)) return fail_value("length %lld exceeds the supported maximum 2^20", (long long)n);
  if (rows > 0 && (reinterpret_cast<uintptr_t>(data) & 15))
    return fail_value("transform buffer must be 16-byte aligned");
  if (variant == MCK_WHT_PARITY) return fwht_parity(data, rows, n, S(st));
  if (variant != MCK_WHT_FAST) return fail_value("unknown transform variant");
  return fwht_fast<float>(data, rows, n, S(st));
}

int mck_fwht_f64(double* data, int64_t rows, int64_t n, void* st) {
  if (!is_pow2(n)) return fail_value("length %lld is not a power of two", (long long)n);
  if (rows < 0) return fail_value("rows must be non-negative");
  if (n > (int64_t(1) << 20)) return fail_value("length %lld exceeds the supported maximum 2^20", (long long)n);
  if (rows > 0 && (reinterpret_cast<uintptr_t>(data) & 15))
    return fail_value("transform buffer must be 16-byte aligned");
  return fwht_fast<double>(data, rows, n, S(st));
}

static int ff_common(const void* tables, int64_t input_dim, int32_t E, double sigma, const float* x,
                     int64_t m, int64_t ldx, int64_t ldo, int64_t min_ld) {
  MCK_TRY(check_spec(input_dim, E, sigma));
  if (!tables) return fail_value("tables buffer is NULL");
  if (m < 0) return fail_value("batch size must be non-negative");
  if (m == 0) return MCK_OK;
  if (ldx < input_dim) return fail_value("input row stride %lld < input_dim %lld", (long long)ldx, (long long)input_dim);
  if (ldo < min_ld) return fail_value("output row stride too small");
  (void)x;
  return MCK_OK;
}

int mck_zhat_f32(const void* tables, int64_t input_dim, int32_t E, double sigma, const float* x,
                 int64_t m, int64_t ldx, const int32_t* row_index, float* z, int64_t ldz,
                 int32_t variant, void* st) {
  const int64_t n = next_pow2(input_dim);
  MCK_TRY(ff_common(tables, input_dim, E, sigma, x, m, ldx, ldz, n * E));
  TablesView tv;
  tables_layout(n, E, (char*)const_cast<void*>(tables), &tv);
  return fastfood_run(tv, (int32_t)input_dim, sigma, x, m, ldx, row_index, false, false, z, ldz,
                      variant, S(st));
}

int mck_features_f32(const void* tables, int64_t input_dim, int32_t E, double sigma, const float* x,
                     int64_t m, int64_t ldx, const int32_t* row_index, int32_t normalize, float* out,
                     int64_t ldo, int32_t variant, void* st) {
  const int64_t n = next_pow2(input_dim);
  MCK_TRY(ff_common(tables, input_dim, E, sigma, x, m, ldx, ldo, 2 * n * E));
  TablesView tv;
  tables_layout(n, E, (char*)const_cast<void*>(tables), &tv);
  return fastfood_run(tv, (int32_t)input_dim, sigma, x, m, ldx, row_index, true, normalize != 0,
                      out, ldo, variant, S(st));
}

int64_t mck_head_scratch_bytes(int64_t m, int64_t F, int32_t C) { return head_scratch_bytes(m, F, C); }

int mck_head_forward(const float* phi, int64_t m, int64_t F, int64_t ld, const double* w,
                     const double* b, int32_t C, const int32_t* labels,
                     const int32_t* label_index, int64_t m_total, double* probs, double* delta,
                     double* loss_sum, int64_t* hits, void* scratch, void* st) {
  if (F < 1 || ld < F) return fail_value("bad feature geometry");
  if (m_total < m) m_total = m;
  return head_forward(phi, m, F, ld, w, b, C, labels, label_index, m_total, probs, delta, loss_sum, hits,
                      scratch, S(st));
}

int mck_head_backward(const float* phi, int64_t m, int64_t F, int64_t ld, const double* delta,
                      int32_t C, double* dw, double* db, void* scratch, void* st) {
  if (F < 1 || ld < F) return fail_value("bad feature geometry");
  return head_backward(phi, m, F, ld, delta, C, dw, db, scratch, S(st));
}

int mck_head_sgd_update(double* w, double* b, const double* dw, const double* db, int64_t F,
                        int32_t C, double lr, double l2, void* st) {
  if (!(lr > 0.0)) return fail_value("learning rate must be positive");
  return head_sgd_update(w, b, dw, db, F, C, lr, l2, S(st));
}

int mck_head_backward_sgd(const float* phi, int64_t m, int64_t F, int64_t ld, const double* delta,
                          int32_t C, double* w, double* b, double lr, double l2, void* scratch,
                          void* st) {
  if (F < 1 || ld < F) return fail_value("bad feature geometry");
  if (!(lr > 0.0)) return fail_value("learning rate must be positive");
  return head_backward_sgd(phi, m, F, ld, delta, C, w, b, lr, l2, scratch, S(st));
}

}  // extern "C"

extern "C" {

int64_t mck_fused_scratch_bytes(int64_t m, int64_t n, int32_t C) {
  if (m < 0 || n < 1 || C < 2) return 0;
  return fused_scratch_bytes(m, n, 1, C, false);
}

int64_t mck_fused_scratch_bytes_ex(int64_t m, int64_t n, int32_t E, int32_t C, int32_t keep_z) {
  if (m < 0 || n < 1 || E < 1 || C < 2) return 0;
  return fused_scratch_bytes(m, n, E, C, keep_z != 0);
}

int mck_fused_forward(const void* tables, int64_t input_dim, int32_t E, double sigma,
                      const float* x, int64_t m, int64_t ldx, const int32_t* row_index,
                      const float* w, const double* b, int32_t C, const int32_t* labels,
                      const int32_t* label_index, int64_t m_total, double* logits, double* probs,
                      double* delta, double* loss_sum, int64_t* hits, void* scratch,
                      int32_t variant, void* st) {
  const int64_t n = next_pow2(input_dim);
  MCK_TRY(ff_common(tables, input_dim, E, sigma, x, m, ldx, 0, 0));
  if (variant < 0 || variant > 7 || (variant & 5) == 5) return fail_value("unknown fused variant %d", variant);
  if (m > 0 && (!w || !b || !delta || !scratch)) return fail_value("NULL argument");
  if (m_total < m) m_total = m;
  TablesView tv;
  tables_layout(n, E, (char*)const_cast<void*>(tables), &tv);
  return fused_forward(tv, (int32_t)input_dim, sigma, x, m, ldx, row_index, w, b, C, labels,
                       label_index, m_total, logits, probs, delta, loss_sum, hits, scratch,
                       variant, S(st));
}

int mck_fused_backward(const void* tables, int64_t input_dim, int32_t E, double sigma,
                       const float* x, int64_t m, int64_t ldx, const int32_t* row_index,
                       const double* delta, int32_t C, float* dw, double* db, float* w, double* b,
                       double lr, double l2, void* scratch, int32_t variant, void* st) {
  const int64_t n = next_pow2(input_dim);
  MCK_TRY(ff_common(tables, input_dim, E, sigma, x, m, ldx, 0, 0));
  if (variant < 0 || variant > 7 || (variant & 5) == 5) return fail_value("unknown fused variant %d", variant);
  if (m > 0 && (!delta || !scratch)) return fail_value("NULL argument");
  if (w && !(lr > 0.0)) return fail_value("learning rate must be positive");
  if (!w && !dw) return fail_value("either w (fused update) or dw is required");
  TablesView tv;
  tables_layout(n, E, (char*)const_cast<void*>(tables), &tv);
  return fused_backward(tv, (int32_t)input_dim, sigma, x, m, ldx, row_index, delta, C, dw, db, w,
                        b, lr, l2, scratch, variant, S(st));
}

int mck_fused_backward_bucket(const void* tables, int64_t input_dim, int32_t E, double sigma,
                              const float* x, int64_t m, int64_t ldx, const int32_t* row_index,
                              const double* delta, int32_t C, int32_t e_begin, int32_t e_count,
                              float* bucket, void* scratch, int32_t variant, void* st) {
  const int64_t n = next_pow2(input_dim);
  MCK_TRY(ff_common(tables, input_dim, E, sigma, x, m, ldx, 0, 0));
  if (e_begin < 0 || e_count < 1 || e_begin + e_count > E)
    return fail_value("block range [%d, %d) outside 0..%d", e_begin, e_begin + e_count, E);
  if (variant < 0 || variant > 7 || (variant & 5) == 5) return fail_value("unknown fused variant %d", variant);
  if (!bucket || (m > 0 && (!delta || !scratch))) return fail_value("NULL argument");
  if (C < 2 || C > 16) return fail_value("num_classes must be in 2..16");
  if (m == 0)
    return check_cuda(cudaMemsetAsync(bucket, 0, (size_t)C * 2 * e_count * n * sizeof(float), S(st)),
                      "bucket clear");
  TablesView tv;
  tables_layout(n, E, (char*)const_cast<void*>(tables), &tv);
  const int64_t nz = (int64_t)e_count * n;
  return fused_backward_range(tv, (int32_t)input_dim, sigma, x, m, ldx, row_index, delta, C, e_begin,
                              e_count, bucket, 2 * nz, 0, nz, nullptr, 0.0, 0.0, scratch, variant, S(st));
}

int mck_fused_bias_grad(const double* delta, int64_t m, int32_t C, double* db, void* st) {
  if (C < 2 || C > 16) return fail_value("num_classes must be in 2..16");
  if (!db || (m > 0 && !delta)) return fail_value("NULL argument");
  if (m == 0) return check_cuda(cudaMemsetAsync(db, 0, (size_t)C * 8, S(st)), "db clear");
  return fused_bias_grad(delta, m, C, db, S(st));
}

int mck_fused_apply_bucket(float* w, int64_t input_dim, int32_t E, int32_t C, int32_t e_begin,
                           int32_t e_count, const float* bucket, double lr, double l2, double* b,
                           const double* db, void* st) {
  if (input_dim < 1 || E < 1) return fail_value("bad spec");
  if (e_begin < 0 || e_count < 1 || e_begin + e_count > E)
    return fail_value("block range [%d, %d) outside 0..%d", e_begin, e_begin + e_count, E);
  if (!(lr > 0.0)) return fail_value("learning rate must be positive");
  if (!w || !bucket || (b && !db)) return fail_value("NULL argument");
  if (C < 2 || C > 16) return fail_value("num_classes must be in 2..16");
  return fused_apply_bucket(w, next_pow2(input_dim), E, C, e_begin, e_count, bucket, lr, l2, b, db, S(st));
}

}  // extern "C"
