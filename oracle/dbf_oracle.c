/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference DBF hot path (/root/reference/pkg/src/dbf, numpy 2.3
 * arithmetic), used by tests/ as a fast checker at full Llama sizes and by bench.py's
 * cpu_baseline leg.  Never linked into or called by the product library.
 *
 * Pinned by tests/test_oracle.py against golden vectors generated from the reference package
 * (tests/golden/make_golden.py).  To be bit-identical with dbf.kernel.sign_matvec, the per-word
 * sums reproduce numpy's float64 add.reduce: for a row segment of n <= 64 values numpy computes
 * 0.0 + pairwise_sum(v), and pairwise_sum uses, for 8 <= n <= 128, eight running accumulators
 * r[j] += v[8i + j], the tree ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and a sequential tail; for
 * n < 8 a plain sequential sum.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static int64_t row_bytes(int64_t cols) { return (cols + 7) / 8; }

/* numpy pairwise_sum for n <= 128 (numpy/_core/src/umath/loops_utils.h.src) */
static double pairwise_sum_small(const double* v, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += v[i];
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = v[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += v[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += v[i];
  return res;
}

/* bitcore.py:72-85.  Returns the row-major index of the first entry with |v| != 1, else -1. */
int64_t dbf_oracle_pack(const double* dense, int64_t rows, int64_t cols, uint8_t* bits) {
  const int64_t rb = row_bytes(cols);
  for (int64_t i = 0; i < rows * cols; ++i)
    if (!(fabs(dense[i]) == 1.0)) return i;
  memset(bits, 0, (size_t)(rows * rb));
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c)
      if (dense[r * cols + c] > 0) bits[r * rb + (c >> 3)] |= (uint8_t)(1u << (c & 7));
  return -1;
}

/* bitcore.py:88-91 */
void dbf_oracle_unpack(const uint8_t* bits, int64_t rows, int64_t cols, double* out) {
  const int64_t rb = row_bytes(cols);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c)
      out[r * cols + c] = ((bits[r * rb + (c >> 3)] >> (c & 7)) & 1) ? 1.0 : -1.0;
}

/* kernel.py:24-45 */
void dbf_oracle_sign_matvec(const uint8_t* bits, int64_t rows, int64_t cols, const double* x,
                            double* out) {
  const int64_t rb = row_bytes(cols);
  const int64_t nwords = (rb + 7) / 8;
  double sel_pos[64], sel_neg[64];
  for (int64_t r = 0; r < rows; ++r) {
    const uint8_t* row = bits + r * rb;
    double pos = 0.0, neg = 0.0;
    for (int64_t w = 0; w < nwords; ++w) {
      const int64_t lo = 8 * w, hi = (8 * w + 8 < rb) ? 8 * w + 8 : rb;
      int64_t ncols = cols - 64 * w;
      if (ncols > (hi - lo) * 8) ncols = (hi - lo) * 8;
      for (int64_t j = 0; j < ncols; ++j) {
        const int64_t c = 64 * w + j;
        const int on = (row[c >> 3] >> (c & 7)) & 1;
        sel_pos[j] = on ? x[c] : 0.0;
        sel_neg[j] = on ? 0.0 : x[c];
      }
      pos += 0.0 + pairwise_sum_small(sel_pos, (int)ncols);
      neg += 0.0 + pairwise_sum_small(sel_neg, (int)ncols);
    }
    out[r] = pos - neg;
  }
}

/* kernel.py:48-62; tmp must hold max(m, k) + k + n doubles. */
void dbf_oracle_forward(const double* X, int64_t batch, const double* a, const uint8_t* A_bits,
                        const double* mid, const uint8_t* B_bits, const double* b, int64_t n,
                        int64_t k, int64_t m, double* out, double* tmp) {
  const int64_t mk = m > k ? m : k;
  double* xs = tmp;          /* max(m, k) */
  double* h = tmp + mk;      /* k */
  double* y = h + k;         /* n */
  for (int64_t i = 0; i < batch; ++i) {
    for (int64_t j = 0; j < m; ++j) xs[j] = X[i * m + j] * b[j];
    dbf_oracle_sign_matvec(B_bits, k, m, xs, h);
    for (int64_t j = 0; j < k; ++j) xs[j] = h[j] * mid[j];
    dbf_oracle_sign_matvec(A_bits, n, k, xs, y);
    for (int64_t j = 0; j < n; ++j) out[i * n + j] = y[j] * a[j];
  }
}
