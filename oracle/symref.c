/*
 * ORACLE — test infrastructure only (never linked into the product).
 *
 * Plain-C restatement of the reference sparse-symbol codec,
 * /root/reference/pkg/src/omniattn/symbols.py:
 *   _compress_groups  symbols.py:39-53  (mixed pool group -> error)
 *   _pack_row         symbols.py:56-62  (MSB-first, zero-padded tail)
 *   encode_cache_mask symbols.py:65-70
 *   encode_skip_mask  symbols.py:73-81  (one byte-aligned row per compressed row)
 *   decode_spatial    symbols.py:163-168
 *   decode_reduction  symbols.py:171-180
 *   decode_run        symbols.py:183-198
 * Pinned against the reference's own golden bytes and reference-generated
 * fixtures (tests/test_oracle_golden.py, tests/golden/).
 */
#include <stdint.h>
#include <string.h>

static int cdiv(int a, int b) { return (a + b - 1) / b; }

/* returns 0, or -1 when a pool group is not uniform (ConsistencyError) */
int ref_encode_cache(const uint8_t* bits, int n, int pool_n, uint8_t* out) {
  int comp = cdiv(n, pool_n);
  memset(out, 0, (size_t)cdiv(comp, 8));
  for (int c = 0; c < comp; ++c) {
    int v0 = bits[c * pool_n] != 0;
    for (int r = c * pool_n; r < n && r < (c + 1) * pool_n; ++r)
      if ((bits[r] != 0) != v0) return -1;
    if (v0) out[c >> 3] |= (uint8_t)(0x80u >> (c & 7));
  }
  return 0;
}

int ref_encode_skip(const uint8_t* bits, int rows, int cols, int pool_n, uint8_t* out) {
  int cr = cdiv(rows, pool_n), cc = cdiv(cols, pool_n), stride = cdiv(cc, 8);
  memset(out, 0, (size_t)cr * stride);
  for (int a = 0; a < cr; ++a)
    for (int b = 0; b < cc; ++b) {
      int v0 = bits[(size_t)(a * pool_n) * cols + b * pool_n] != 0;
      for (int r = a * pool_n; r < rows && r < (a + 1) * pool_n; ++r)
        for (int c = b * pool_n; c < cols && c < (b + 1) * pool_n; ++c)
          if ((bits[(size_t)r * cols + c] != 0) != v0) return -1;
      if (v0) out[(size_t)a * stride + (b >> 3)] |= (uint8_t)(0x80u >> (b & 7));
    }
  return 0;
}

int ref_decode_spatial(const uint8_t* s_c, int pool_n, int i) {
  int c = i / pool_n;
  return (s_c[c >> 3] >> (7 - (c & 7))) & 1;
}

int ref_decode_reduction(const uint8_t* s_s, int cols, int pool_n, int i, int j) {
  int stride = cdiv(cdiv(cols, pool_n), 8);
  int ci = i / pool_n, cj = j / pool_n;
  return (s_s[(size_t)ci * stride + (cj >> 3)] >> (7 - (cj & 7))) & 1;
}

/* decode_run: one compressed row expanded to `cols` per-block bits */
void ref_decode_run(const uint8_t* s_s, int cols, int pool_n, int comp_row, uint8_t* out) {
  int stride = cdiv(cdiv(cols, pool_n), 8);
  const uint8_t* row = s_s + (size_t)comp_row * stride;
  for (int j = 0; j < cols; ++j) {
    int cj = j / pool_n;
    out[j] = (row[cj >> 3] >> (7 - (cj & 7))) & 1;
  }
}
