// Text graph ingestion on device (graphs.py:96-202) and the binary CSR cache.
//
// load_edge_list's per-line work -- split on whitespace, Python int()
// parsing, comment/blank skipping, range checks -- runs as sm_100a kernels
// over the file's bytes in HBM:
//   k_count_ends / k_write_ends  line terminators ("\n", "\r\n", lone "\r":
//                                universal newlines) -> line end offsets,
//                                via a tile-count scan
//   k_parse_lines<fmt>           thread per line: classify, tokenise, parse
//                                both ids; the first error (lowest line) wins
//                                through one 64-bit atomicMin
//   k_compact_edges              edge lines -> the (m, 2) edge array, in
//                                file order (flag scan)
// The Matrix Market header and size line are read on the host (two lines);
// the device parses the coordinate entries that follow.  The parsed edges
// stay in HBM for the CSR build (bfb_graph_from_parsed) or are copied out.
// Error messages are formatted by the caller from (line, code, byte range),
// so they are the reference's ParseError texts verbatim.
#include <cstdio>
#include <cstring>
#include <vector>

#include "bfb_device.cuh"
#include "bfb_internal.cuh"

namespace bfb {
namespace {

constexpr int kBlock = 256;
constexpr int kBytesPerThread = 16;
constexpr int64_t kByteTile = (int64_t)kBlock * kBytesPerThread;
constexpr uint64_t kMaxVid = 0xFFFFFFFFull;

__host__ __device__ __forceinline__ bool is_ws(unsigned char c) {
  // str.isspace() over ASCII: \t \n \v \f \r, \x1c-\x1f and space
  return (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x20);
}

// A line terminator ends at byte i: '\n', or (universal newlines, nl = 0) a
// '\r' not followed by '\n'.  nl = 1: '\n' only (an io.StringIO source).
__device__ __forceinline__ bool line_end_at(const unsigned char* b, int64_t i, int64_t len, int nl) {
  const unsigned char c = b[i];
  return c == '\n' || (nl == 0 && c == '\r' && (i + 1 >= len || b[i + 1] != '\n'));
}

__global__ void __launch_bounds__(kBlock) k_count_ends(const unsigned char* b, int64_t len, int nl,
                                                       uint32_t* tile_counts) {
  const int64_t base = (int64_t)blockIdx.x * kByteTile + (int64_t)threadIdx.x * kBytesPerThread;
  int64_t c = 0;
  for (int k = 0; k < kBytesPerThread; ++k)
    if (base + k < len && line_end_at(b, base + k, len, nl)) ++c;
  __shared__ int64_t red[kBlock / 32];
  c = block_sum_i64(c, red);
  if (threadIdx.x == 0) tile_counts[blockIdx.x] = (uint32_t)c;
}

__global__ void __launch_bounds__(kBlock) k_write_ends(const unsigned char* b, int64_t len, int nl,
                                                       const int64_t* tile_pre, int64_t* ends) {
  const int64_t base = (int64_t)blockIdx.x * kByteTile + (int64_t)threadIdx.x * kBytesPerThread;
  int64_t c = 0;
  for (int k = 0; k < kBytesPerThread; ++k)
    if (base + k < len && line_end_at(b, base + k, len, nl)) ++c;
  __shared__ int64_t wsum[33];
  int64_t total;
  int64_t pos = tile_pre[blockIdx.x] + block_exclusive_i64(c, wsum, &total);
  for (int k = 0; k < kBytesPerThread; ++k)
    if (base + k < len && line_end_at(b, base + k, len, nl)) ends[pos++] = base + k;
}

}  // namespace

// Python int() on one ASCII token: [+-]? digit ("_"? digit)*.  *mag saturates
// above 2^63 (only "> MAX_VID" matters); *neg = '-' sign with a nonzero value.
__host__ __device__ bool parse_py_int(const unsigned char* p, const unsigned char* e, uint64_t* mag,
                                      bool* neg) {
  bool minus = false;
  if (p < e && (*p == '+' || *p == '-')) {
    minus = *p == '-';
    ++p;
  }
  if (p >= e) return false;
  uint64_t v = 0;
  bool prev_digit = false;
  for (; p < e; ++p) {
    const unsigned char c = *p;
    if (c >= '0' && c <= '9') {
      v = v > (1ull << 59) ? (1ull << 63) : v * 10 + (c - '0');
      prev_digit = true;
    } else if (c == '_' && prev_digit && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  *mag = v;
  *neg = minus && v != 0;
  return true;
}

namespace {

// Parse outcome codes (decoded into the reference's ParseError texts by the
// Python layer, paper_2103_13577_b200/graphs.py).
enum : int {
  kPkSkip = 0,      // blank or comment line
  kPkEdge = 1,      // a parsed edge
  kErrTokens = 2,   // edges: "expected 'src dst', got ..."
  kErrNonInt = 3,   // edges: "non-integer vertex id in ..."
  kErrNeg = 4,      // edges: "negative vertex id in ..."
  kErrRangeU = 5,   // edges: "vertex id {u} exceeds the representable range"
  kErrRangeV = 6,   // edges: same for v
  kErrEntry = 7,    // mtx: "expected coordinate entry, got ..."
  kErrMtxInt = 8,   // mtx: "non-integer coordinate in ..."
  kErrOutside = 9,  // mtx: "coordinate (i, j) outside RxC"
};

struct ParseOut {
  int code;
  uint32_t u, v;
};

// fmt 0 = "edges" (graphs.py:109-134), 1 = "mtx" coordinate entries (graphs.py:165-180).
__device__ ParseOut parse_line(const unsigned char* s, const unsigned char* e, int fmt,
                               int64_t rows, int64_t cols) {
  ParseOut o{kPkSkip, 0, 0};
  while (s < e && is_ws(*s)) ++s;
  while (e > s && is_ws(e[-1])) --e;
  if (s == e) return o;
  if (*s == '%' || (fmt == 0 && *s == '#')) return o;
  const unsigned char* tb[2];
  const unsigned char* te[2];
  int ntok = 0;
  const unsigned char* p = s;
  while (p < e) {
    const unsigned char* q = p;
    while (q < e && !is_ws(*q)) ++q;
    if (ntok < 2) {
      tb[ntok] = p;
      te[ntok] = q;
    }
    ++ntok;
    if (ntok > 2) break;
    p = q;
    while (p < e && is_ws(*p)) ++p;
  }
  uint64_t a = 0, b = 0;
  bool na = false, nb = false;
  if (fmt == 0) {
    if (ntok != 2) return {kErrTokens, 0, 0};
    const bool ok1 = parse_py_int(tb[0], te[0], &a, &na);
    const bool ok2 = parse_py_int(tb[1], te[1], &b, &nb);
    if (!ok1 || !ok2) return {kErrNonInt, 0, 0};
    if (na || nb) return {kErrNeg, 0, 0};
    if (a > kMaxVid) return {kErrRangeU, 0, 0};
    if (b > kMaxVid) return {kErrRangeV, 0, 0};
    return {kPkEdge, (uint32_t)a, (uint32_t)b};
  }
  if (ntok < 2) return {kErrEntry, 0, 0};
  const bool ok1 = parse_py_int(tb[0], te[0], &a, &na);
  const bool ok2 = parse_py_int(tb[1], te[1], &b, &nb);
  if (!ok1 || !ok2) return {kErrMtxInt, 0, 0};
  if (na || nb || a < 1 || b < 1 || a > (uint64_t)rows || b > (uint64_t)cols)
    return {kErrOutside, 0, 0};
  return {kPkEdge, (uint32_t)(a - 1), (uint32_t)(b - 1)};
}

__global__ void k_parse_lines(const unsigned char* b, const int64_t* ends, int64_t nlines, int fmt,
                              int64_t rows, int64_t cols, int64_t line0, uint32_t* flag,
                              uint2* edge, unsigned long long* first_err,
                              unsigned long long* max_id) {
  uint32_t mx = 0;
  bool any = false;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nlines;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = k ? ends[k - 1] + 1 : 0;
    const ParseOut o = parse_line(b + s, b + ends[k], fmt, rows, cols);
    flag[k] = o.code == kPkEdge;
    if (o.code == kPkEdge) {
      edge[k] = make_uint2(o.u, o.v);
      mx = max(mx, max(o.u, o.v));
      any = true;
    } else if (o.code != kPkSkip) {
      atomicMin(first_err, ((unsigned long long)(line0 + k + 1) << 8) | (unsigned long long)o.code);
    }
  }
  if (any) atomicMax(max_id, (unsigned long long)mx + 1);
}

__global__ void k_compact_edges(const uint32_t* flag, const uint2* edge, const int64_t* pos,
                                int64_t nlines, uint2* out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nlines;
       k += (int64_t)gridDim.x * blockDim.x)
    if (flag[k]) out[pos[k]] = edge[k];
}

unsigned grid_of(int64_t work, int block, int sms) {
  int64_t g = (work + block - 1) / block;
  const int64_t cap = (int64_t)sms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace

int parse_text(bfb_ctx* ctx, const char* data, int64_t len, int fmt, int nl, int64_t line0,
               int64_t rows, int64_t cols, bfb_parse_result* res) {
  std::memset(res, 0, sizeof(*res));
  ctx->parsed.release();
  ctx->parsed_m = 0;
  cudaStream_t s = ctx->stream;
  // bytes + a terminating '\n' unless the text already ends a line
  const bool term = len > 0 && (data[len - 1] == '\n' || (nl == 0 && data[len - 1] == '\r'));
  const int64_t blen = len + (len > 0 && !term ? 1 : 0);
  DevBuf<unsigned char> buf;
  BFB_TRY(buf.alloc(blen + 1));
  if (len) BFB_CUDA(cudaMemcpyAsync(buf.p, data, len, cudaMemcpyHostToDevice, s));
  if (blen > len) BFB_CUDA(cudaMemsetAsync(buf.p + len, '\n', 1, s));
  const int64_t ntiles = (blen + kByteTile - 1) / kByteTile;
  DevBuf<uint32_t> tcnt;
  DevBuf<int64_t> tpre, tmp;
  BFB_TRY(tcnt.alloc(ntiles + 1));
  BFB_TRY(tpre.alloc(ntiles + 1));
  BFB_TRY(tmp.alloc(scan_tmp_words(ntiles + 1) + 1));
  int64_t nlines = 0;
  if (ntiles) {
    k_count_ends<<<(unsigned)ntiles, kBlock, 0, s>>>(buf.p, blen, nl, tcnt.p);
    BFB_CUDA(cudaMemsetAsync(tcnt.p + ntiles, 0, sizeof(uint32_t), s));
    BFB_TRY(scan_u32_to_i64(tcnt.p, ntiles + 1, tpre.p, tmp.p, s));
    BFB_CUDA(cudaMemcpyAsync(&nlines, tpre.p + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    BFB_CUDA(cudaStreamSynchronize(s));
  }
  DevBuf<int64_t> ends, pos, ptmp;
  DevBuf<uint32_t> flag;
  DevBuf<uint2> edge;
  DevBuf<unsigned long long> scal;  // first error, max id + 1
  BFB_TRY(ends.alloc(nlines + 1));
  BFB_TRY(flag.alloc(nlines + 1));
  BFB_TRY(edge.alloc(nlines + 1));
  BFB_TRY(pos.alloc(nlines + 1));
  BFB_TRY(ptmp.alloc(scan_tmp_words(nlines + 1) + 1));
  BFB_TRY(scal.alloc(2));
  const unsigned long long init[2] = {~0ull, 0ull};
  BFB_CUDA(cudaMemcpyAsync(scal.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (nlines) {
    k_write_ends<<<(unsigned)ntiles, kBlock, 0, s>>>(buf.p, blen, nl, tpre.p, ends.p);
    k_parse_lines<<<grid_of(nlines, 256, ctx->num_sms), 256, 0, s>>>(
        buf.p, ends.p, nlines, fmt, rows, cols, line0, flag.p, edge.p, scal.p, scal.p + 1);
  }
  unsigned long long h[2] = {~0ull, 0ull};
  BFB_CUDA(cudaMemcpyAsync(h, scal.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  BFB_CUDA(cudaGetLastError());
  res->num_lines = nlines;
  if (h[0] != ~0ull) {
    const int64_t line_no = (int64_t)(h[0] >> 8);
    const int64_t k = line_no - line0 - 1;
    res->err_line = line_no;
    res->err_code = (int32_t)(h[0] & 0xFF);
    int64_t se[2] = {0, 0};
    if (k > 0) BFB_CUDA(cudaMemcpy(&se[0], ends.p + k - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    BFB_CUDA(cudaMemcpy(&se[1], ends.p + k, sizeof(int64_t), cudaMemcpyDeviceToHost));
    res->err_begin = k > 0 ? se[0] + 1 : 0;
    res->err_end = std::min(se[1], len);
    return fail(BFB_ERR_PARSE, "parse error at line " + std::to_string(line_no));
  }
  res->max_id_plus1 = (int64_t)h[1];
  // compaction of the edge lines, in file order
  BFB_CUDA(cudaMemsetAsync(flag.p + nlines, 0, sizeof(uint32_t), s));
  BFB_TRY(scan_u32_to_i64(flag.p, nlines + 1, pos.p, ptmp.p, s));
  int64_t m = 0;
  BFB_CUDA(cudaMemcpyAsync(&m, pos.p + nlines, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  BFB_CUDA(cudaStreamSynchronize(s));
  BFB_TRY(ctx->parsed.alloc(m + 1));
  if (m)
    k_compact_edges<<<grid_of(nlines, 256, ctx->num_sms), 256, 0, s>>>(flag.p, edge.p, pos.p,
                                                                       nlines, ctx->parsed.p);
  BFB_CUDA(cudaStreamSynchronize(s));
  BFB_CUDA(cudaGetLastError());
  ctx->parsed_m = m;
  res->num_edges = m;
  return BFB_OK;
}

int parsed_copy(bfb_ctx* ctx, uint32_t* out) {
  if (!ctx->parsed.p) return fail(BFB_ERR_STATE, "no parsed edges");
  if (ctx->parsed_m)
    BFB_CUDA(cudaMemcpy(out, ctx->parsed.p, ctx->parsed_m * sizeof(uint2), cudaMemcpyDeviceToHost));
  return BFB_OK;
}

// write_edge_list (graphs.py:205-209): 'u v\n' per edge, byte-identical to
// the reference's f-string output.
int write_edge_list(const char* path, const uint32_t* edges, int64_t m) {
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(BFB_ERR_IO, std::string("cannot open ") + path + " for writing");
  std::vector<char> out((size_t)1 << 24);
  size_t at = 0;
  bool ok = true;
  auto put = [&](uint32_t x) {
    char t[10];
    int k = 0;
    do {
      t[k++] = (char)('0' + x % 10);
      x /= 10;
    } while (x);
    while (k) out[at++] = t[--k];
  };
  for (int64_t i = 0; i < m && ok; ++i) {
    put(edges[2 * i]);
    out[at++] = ' ';
    put(edges[2 * i + 1]);
    out[at++] = '\n';
    if (at > out.size() - 32) {
      ok = std::fwrite(out.data(), 1, at, f) == at;
      at = 0;
    }
  }
  if (ok && at) ok = std::fwrite(out.data(), 1, at, f) == at;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return fail(BFB_ERR_IO, std::string("writing ") + path + " failed");
  return BFB_OK;
}

// ---------------------------------------------------------- CSR cache -----
// File: "BFBCSR01", int64 n, int64 m, int64 offsets[n+1], uint32 adjacency[m].
static const char kCsrMagic[8] = {'B', 'F', 'B', 'C', 'S', 'R', '0', '1'};

int graph_save(bfb_ctx* ctx, const char* path) {
  if (!ctx->g.valid) return fail(BFB_ERR_STATE, "no graph loaded");
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(BFB_ERR_IO, std::string("cannot open ") + path + " for writing");
  const int64_t n = ctx->g.n, m = ctx->g.m;
  const size_t chunk = (size_t)1 << 26;
  std::vector<unsigned char> host(chunk * 8);
  bool ok = std::fwrite(kCsrMagic, 1, 8, f) == 8 && std::fwrite(&n, 8, 1, f) == 1 &&
            std::fwrite(&m, 8, 1, f) == 1;
  auto dump = [&](const void* dev, size_t bytes) {
    for (size_t o = 0; ok && o < bytes; o += host.size()) {
      const size_t k = std::min(host.size(), bytes - o);
      if (cudaMemcpy(host.data(), (const unsigned char*)dev + o, k, cudaMemcpyDeviceToHost) != cudaSuccess) {
        ok = false;
        break;
      }
      ok = std::fwrite(host.data(), 1, k, f) == k;
    }
  };
  dump(ctx->g.offsets.p, (size_t)(n + 1) * sizeof(int64_t));
  dump(ctx->g.adj.p, (size_t)m * sizeof(uint32_t));
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return fail(BFB_ERR_IO, std::string("writing ") + path + " failed");
  return BFB_OK;
}

int graph_load(bfb_ctx* ctx, const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(BFB_ERR_IO, std::string("cannot open ") + path);
  char magic[8];
  int64_t n = -1, m = -1;
  bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, kCsrMagic, 8) == 0 &&
            std::fread(&n, 8, 1, f) == 1 && std::fread(&m, 8, 1, f) == 1 && n >= 0 && m >= 0 &&
            n <= ((int64_t)1 << 32);
  if (!ok) {
    std::fclose(f);
    return fail(BFB_ERR_IO, std::string(path) + " is not a BFBCSR01 graph file");
  }
  std::vector<int64_t> off((size_t)n + 1);
  std::vector<uint32_t> adj((size_t)m);
  ok = std::fread(off.data(), 8, off.size(), f) == off.size() &&
       std::fread(adj.data(), 4, adj.size(), f) == adj.size();
  std::fclose(f);
  if (!ok) return fail(BFB_ERR_IO, std::string(path) + " is truncated");
  if (off[0] != 0 || off[n] != m) return fail(BFB_ERR_IO, std::string(path) + " has inconsistent offsets");
  return load_csr(ctx, n, m, off.data(), adj.data());
}

}  // namespace bfb
