// bm_io.cpp — graph files on the host (include/bmatch_b200_io.h): Matrix
// Market ingest and export, and the binary CSC container. Not on the matching
// hot path: this is the step before
// bm_upload_csc.
//
// Matrix Market ingest follows read_matrix_market (matrix_market.cpp:29-99)
// rule for rule, but runs on every host core. The header is parsed serially.
// The data section is memory-mapped and split into line-aligned chunks that
// are scanned three times:
//   1. validate: count lines, data lines and edges per chunk, and record each
//      chunk's first error;
//   2. count column degrees (build_csc pass 1);
//   3. scatter rows, then sort and de-duplicate each column (build_csc).
// Between 1 and 2 a serial walk over the chunk summaries turns the per-chunk
// findings into the error the reference's line-at-a-time reader reports
// first, with its line number.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cctype>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bm_host_util.hpp"
#include "bmatch_b200_io.h"

namespace {

using namespace bm_host;

bm_status parse_fail(int64_t line, const std::string& msg, int64_t* err_line) {
  if (err_line) *err_line = line;
  bm_internal_set_error("line " + std::to_string(line) + ": " + msg);  // ParseError's what()
  return BM_ERR_PARSE;
}

bm_status io_fail(const std::string& msg) { return hfail(BM_ERR_IO, msg); }

// isspace() in the "C" locale, which is what istream >> uses here.
inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f' || c == '\n'; }

// A line as std::getline yields it: [b, e) without the '\n'.
struct Line {
  const char* b;
  const char* e;
};

// Calls fn(Line) for every line in [b, e) where b is a line start. Returns
// the number of lines: one per '\n', plus a final unterminated one.
template <typename F>
inline void for_lines(const char* b, const char* e, F&& fn) {
  while (b < e) {
    const char* q = static_cast<const char*>(std::memchr(b, '\n', (size_t)(e - b)));
    if (!q) q = e;
    fn(Line{b, q});
    b = q + 1;
  }
}

// The reference skips `line.empty() || line[0] == '%' || is_blank(line)`.
inline bool skippable(const Line& l) {
  if (l.b == l.e || *l.b == '%') return true;
  for (const char* p = l.b; p < l.e; ++p)
    if (!is_ws(*p)) return false;
  return true;
}

// istream >> long long: leading whitespace, optional sign, at least one
// decimal digit; overflow fails.
inline bool next_ll(const char*& p, const char* e, long long& v) {
  while (p < e && is_ws(*p)) ++p;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p >= e || *p < '0' || *p > '9') return false;
  unsigned long long acc = 0;
  const unsigned long long lim = neg ? (unsigned long long)LLONG_MAX + 1 : (unsigned long long)LLONG_MAX;
  while (p < e && *p >= '0' && *p <= '9') {
    const unsigned d = (unsigned)(*p++ - '0');
    if (acc > (lim - d) / 10) return false;
    acc = acc * 10 + d;
  }
  v = neg ? (long long)(0ULL - acc) : (long long)acc;
  return true;
}

// istream >> std::string: the next whitespace-delimited token ("" at end).
inline std::string next_tok(const char*& p, const char* e) {
  while (p < e && is_ws(*p)) ++p;
  const char* b = p;
  while (p < e && !is_ws(*p)) ++p;
  return std::string(b, p);
}

std::string lower(std::string s) {
  for (char& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

struct Header {
  bm_mm_header h{};
  int64_t data_begin = 0;  // byte offset of the first line after the size line
  int64_t size_line = 0;   // 1-based line number of the size line
};

// Banner and size line (matrix_market.cpp:33-69).
bm_status parse_header(const char* buf, int64_t len, Header& H, int64_t* err_line) {
  if (len <= 0) return parse_fail(1, "empty stream", err_line);
  const char* end = buf + len;
  const char* q = static_cast<const char*>(std::memchr(buf, '\n', (size_t)len));
  if (!q) q = end;
  const char* p = buf;
  const std::string banner = next_tok(p, q);
  const std::string object = lower(next_tok(p, q)), format = lower(next_tok(p, q));
  const std::string field = lower(next_tok(p, q)), symmetry = lower(next_tok(p, q));
  if (banner != "%%MatrixMarket") return parse_fail(1, "missing %%MatrixMarket banner", err_line);
  if (object != "matrix") return parse_fail(1, "unsupported object '" + object + "'", err_line);
  if (format != "coordinate") return parse_fail(1, "unsupported format '" + format + "'", err_line);
  if (field != "pattern" && field != "real" && field != "integer")
    return parse_fail(1, "unsupported field '" + field + "'", err_line);
  if (symmetry != "general" && symmetry != "symmetric")
    return parse_fail(1, "unsupported symmetry '" + symmetry + "'", err_line);
  H.h.symmetric = symmetry == "symmetric";
  H.h.field = field == "pattern" ? 0 : field == "real" ? 1 : 2;

  long long rows = -1, cols = -1, entries = -1, lineno = 1;
  const char* pos = q < end ? q + 1 : end;
  while (pos < end) {  // std::getline succeeds while characters remain
    const char* nl = static_cast<const char*>(std::memchr(pos, '\n', (size_t)(end - pos)));
    if (!nl) nl = end;
    const Line l{pos, nl};
    pos = nl < end ? nl + 1 : end;
    ++lineno;
    if (skippable(l)) continue;
    const char* t = l.b;
    if (!next_ll(t, l.e, rows) || !next_ll(t, l.e, cols) || !next_ll(t, l.e, entries))
      return parse_fail(lineno, "malformed size line", err_line);
    break;
  }
  if (rows < 0) return parse_fail(lineno + 1, "missing size line", err_line);
  if (rows > INT_MAX || cols > INT_MAX) return parse_fail(lineno, "dimensions too large", err_line);
  // The reference goes on to reserve/assign with these (UB or length_error); reject cleanly.
  if (cols < 0) return hfail(BM_ERR_INVALID_ARG, "negative column count in the size line");
  if (entries < 0) return hfail(BM_ERR_INVALID_ARG, "negative entry count in the size line");
  H.h.nrows = (int32_t)rows;
  H.h.ncols = (int32_t)cols;
  H.h.entries = entries;
  H.h.capacity = H.h.symmetric ? 2 * entries : entries;
  H.data_begin = pos - buf;
  H.size_line = lineno;
  return BM_OK;
}

// What pass 1 learns about one chunk.
struct ChunkScan {
  int64_t b = 0, e = 0;         // byte range [b, e), both line starts
  int64_t lines = 0, data = 0;  // lines, non-skippable lines
  int64_t edges = 0;            // edges the valid entries emit
  int64_t err_line = -1;        // chunk-local 0-based line of the first parse error
  int64_t err_data = 0;         // its data-line index within the chunk
  std::string err;
  int64_t rng_edge = -1;        // chunk-local index of the first out-of-range edge (from_edge_list)
  std::string rng;
};

struct Parsed {
  long long i, j;
};

// One entry line: 1-based (row i, column j) checked against the header
// (matrix_market.cpp:74-88). Returns "" or the reference's message.
inline const char* parse_entry(const Line& l, const Header& H, Parsed& out, std::string& msg) {
  const char* t = l.b;
  if (!next_ll(t, l.e, out.i) || !next_ll(t, l.e, out.j)) return "malformed entry";
  if (out.i < 1 || out.i > H.h.nrows) {
    msg = "row index " + std::to_string(out.i) + " outside [1, " + std::to_string(H.h.nrows) + "]";
    return msg.c_str();
  }
  if (out.j < 1 || out.j > H.h.ncols) {
    msg = "column index " + std::to_string(out.j) + " outside [1, " + std::to_string(H.h.ncols) + "]";
    return msg.c_str();
  }
  return "";
}

bm_status parse_mm(const char* buf, int64_t len, int threads, int64_t capacity, int64_t* cxadj, int32_t* cadj,
                   int64_t* nedges, int64_t* err_line) {
  Header H;
  if (bm_status s = parse_header(buf, len, H, err_line)) return s;
  if (!cxadj || !nedges || (capacity > 0 && !cadj)) return hfail(BM_ERR_INVALID_ARG, "null output buffer");
  threads = resolve_threads(threads);
  const int nc = H.h.ncols, nr = H.h.nrows;
  const bool mirror = H.h.symmetric;

  // Line-aligned chunks of about 8 MB (BM_MM_CHUNK bytes: tests use tiny
  // chunks to put many boundaries into small files).
  const int64_t dlen = len - H.data_begin;
  const char* env = std::getenv("BM_MM_CHUNK");
  const int64_t target = env && std::atoll(env) > 0 ? std::atoll(env) : 8LL << 20;
  const int64_t nominal = std::max<int64_t>(1, (dlen + target - 1) / target);
  std::vector<int64_t> starts{H.data_begin};
  for (int64_t k = 1; k < nominal; ++k) {
    int64_t s = H.data_begin + dlen * k / nominal;
    if (s <= starts.back()) continue;
    if (buf[s - 1] != '\n') {
      const char* nl = static_cast<const char*>(std::memchr(buf + s, '\n', (size_t)(len - s)));
      s = nl ? nl + 1 - buf : len;
    }
    if (s > starts.back() && s < len) starts.push_back(s);
  }
  std::vector<ChunkScan> ch(starts.size());
  for (size_t k = 0; k < ch.size(); ++k) {
    ch[k].b = starts[k];
    ch[k].e = k + 1 < starts.size() ? starts[k + 1] : len;
  }

  // Pass 1: validate.
  parallel_chunks((long long)ch.size(), threads, [&](long long k) {
    ChunkScan& c = ch[k];
    std::string msg;
    for_lines(buf + c.b, buf + c.e, [&](const Line& l) {
      const int64_t ln = c.lines++;
      if (skippable(l)) return;
      const int64_t d = c.data++;
      if (c.err_line >= 0) return;  // only counting after the chunk's first error
      Parsed pe;
      const char* m = parse_entry(l, H, pe, msg);
      if (*m) {
        c.err_line = ln;
        c.err_data = d;
        c.err = m;
        return;
      }
      ++c.edges;  // (c = j-1, r = i-1) is in range once the entry is
      if (mirror && pe.i != pe.j) {
        // The mirrored edge (c = i-1, r = j-1) can leave a non-square matrix;
        // from_edge_list rejects it (csr_graph.cpp:12-24).
        if (c.rng_edge < 0 && (pe.i - 1 >= nc || pe.j - 1 >= nr)) {
          c.rng_edge = c.edges;
          const std::string cr = " (c=" + std::to_string(pe.i - 1) + ", r=" + std::to_string(pe.j - 1) + "): ";
          c.rng = pe.i - 1 >= nc ? cr + "column index outside [0, " + std::to_string(nc) + ")"
                                 : cr + "row index outside [0, " + std::to_string(nr) + ")";
        }
        ++c.edges;
      }
    });
  });

  // The first error in file order, as the line-at-a-time reader meets it.
  const int64_t E = H.h.entries;
  int64_t line_base = H.size_line, data_base = 0;
  for (const ChunkScan& c : ch) {
    if (c.err_line >= 0 && data_base + c.err_data < E) return parse_fail(line_base + 1 + c.err_line, c.err, err_line);
    if (data_base + c.data > E) {
      // The (E+1)-th data line is the first one read after the declared entries.
      int64_t want = E - data_base, ln = 0, found = -1;
      for_lines(buf + c.b, buf + c.e, [&](const Line& l) {
        const int64_t me = ln++;
        if (found >= 0 || skippable(l)) return;
        if (want-- == 0) found = me;
      });
      return parse_fail(line_base + 1 + found,
                        "entry count mismatch: data after the declared " + std::to_string(E) + " entries", err_line);
    }
    line_base += c.lines;
    data_base += c.data;
  }
  if (data_base < E)
    return parse_fail(line_base + 1,
                      "entry count mismatch: expected " + std::to_string(E) + ", found " + std::to_string(data_base),
                      err_line);
  int64_t edge_base = 0;
  for (const ChunkScan& c : ch) {
    if (c.rng_edge >= 0) return hfail(BM_ERR_INVALID_ARG, "edge " + std::to_string(edge_base + c.rng_edge) + c.rng);
    edge_base += c.edges;
  }
  if (edge_base > capacity) return hfail(BM_ERR_INVALID_ARG, "capacity below the header's entry count");

  // Passes 2-3: the shared sorted + de-duplicated CSC builder.
  auto produce = [&](long long k, auto&& emit) {
    std::string unused;
    for_lines(buf + ch[k].b, buf + ch[k].e, [&](const Line& l) {
      if (skippable(l)) return;
      const char* t = l.b;
      long long i = 0, j = 0;
      next_ll(t, l.e, i);
      next_ll(t, l.e, j);
      emit((int)(j - 1), (int)(i - 1));
      if (mirror && i != j) emit((int)(i - 1), (int)(j - 1));
    });
  };
  if (err_line) *err_line = 0;
  return build_csc(nc, nr, (long long)ch.size(), threads, capacity, produce, cxadj, cadj, nedges);
}

// Read-only mapping of a whole file.
struct Mapped {
  const char* p = nullptr;
  int64_t n = 0;
  int fd = -1;
  ~Mapped() {
    if (p && n > 0) munmap(const_cast<char*>(p), (size_t)n);
    if (fd >= 0) close(fd);
  }
  bm_status open_file(const char* path) {
    if (!path) return hfail(BM_ERR_INVALID_ARG, "null path");
    fd = ::open(path, O_RDONLY);
    if (fd < 0) return io_fail(std::string("cannot open '") + path + "'");
    struct stat st;
    if (fstat(fd, &st) != 0) return io_fail(std::string("cannot stat '") + path + "'");
    n = (int64_t)st.st_size;
    if (n == 0) return BM_OK;
    void* m = mmap(nullptr, (size_t)n, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) return io_fail(std::string("cannot map '") + path + "'");
    madvise(m, (size_t)n, MADV_SEQUENTIAL);
    p = static_cast<const char*>(m);
    return BM_OK;
  }
};

// ---- writers -------------------------------------------------------------

inline char* put_u64(char* o, unsigned long long v) {
  char tmp[24];
  int k = 0;
  do {
    tmp[k++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  while (k) *o++ = tmp[--k];
  return o;
}

// Parallel pwrite / pread of one contiguous region in 64 MB pieces.
bm_status pio(int fd, bool write, char* mem, int64_t bytes, int64_t off, int threads) {
  const int64_t piece = 64LL << 20;
  const long long np = (bytes + piece - 1) / piece;
  std::atomic<bool> ok{true};
  parallel_chunks(np, threads, [&](long long k) {
    int64_t done = k * piece;
    const int64_t stop = std::min<int64_t>(bytes, done + piece);
    while (done < stop && ok.load(std::memory_order_relaxed)) {
      const ssize_t r = write ? pwrite(fd, mem + done, (size_t)(stop - done), off + done)
                              : pread(fd, mem + done, (size_t)(stop - done), off + done);
      if (r <= 0) {
        ok = false;
        return;
      }
      done += r;
    }
  });
  return ok ? BM_OK : io_fail(write ? "short write" : "short read");
}

struct CscHeader {
  char magic[8];
  int32_t nc, nr;
  int64_t nedges;
  uint64_t checksum;
  uint64_t reserved;
};
static_assert(sizeof(CscHeader) == 40, "binary CSC header is 40 bytes");
constexpr char kMagic[8] = {'B', 'M', 'C', 'S', 'C', '0', '0', '1'};

inline uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  return x ^ (x >> 33);
}

// Order-dependent checksum of the two arrays: per-8 MB-block hashes (computed
// in parallel) folded in block order.
uint64_t csc_checksum(int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj, int64_t ne, int threads) {
  struct Region {
    const unsigned char* p;
    int64_t n;
  };
  const Region reg[2] = {{reinterpret_cast<const unsigned char*>(cxadj), 8 * ((int64_t)nc + 1)},
                         {reinterpret_cast<const unsigned char*>(cadj), 4 * ne}};
  const int64_t blk = 8LL << 20;
  std::vector<std::pair<int, int64_t>> blocks;
  for (int r = 0; r < 2; ++r)
    for (int64_t o = 0; o < reg[r].n; o += blk) blocks.emplace_back(r, o);
  std::vector<uint64_t> hs(blocks.size());
  parallel_chunks((long long)blocks.size(), threads, [&](long long k) {
    const Region& R = reg[blocks[k].first];
    const int64_t o = blocks[k].second, n = std::min(blk, R.n - o);
    uint64_t h = 0x9e3779b97f4a7c15ULL ^ (uint64_t)k;
    int64_t i = 0;
    for (; i + 8 <= n; i += 8) {
      uint64_t w;
      std::memcpy(&w, R.p + o + i, 8);
      h = (h ^ w) * 0x100000001b3ULL;
      h ^= h >> 29;
    }
    for (; i < n; ++i) h = (h ^ R.p[o + i]) * 0x100000001b3ULL;
    hs[k] = mix64(h ^ (uint64_t)n);
  });
  uint64_t h = mix64(((uint64_t)(uint32_t)nc << 32) ^ (uint32_t)nr) ^ mix64((uint64_t)ne);
  for (uint64_t x : hs) h = mix64(h ^ x) + 0x632be59bd9b4e019ULL;
  return h;
}

}  // namespace

extern "C" {

bm_status bm_mm_parse_info(const char* text, int64_t length, bm_mm_header* header, int64_t* err_line) {
  if (!header || (!text && length > 0) || length < 0) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  Header H;
  if (bm_status s = parse_header(text, length, H, err_line)) return s;
  *header = H.h;
  return BM_OK;
}

bm_status bm_mm_parse(const char* text, int64_t length, int32_t threads, int64_t capacity, int64_t* cxadj,
                      int32_t* cadj, int64_t* nedges, int64_t* err_line) {
  if ((!text && length > 0) || length < 0) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  return parse_mm(text, length, threads, capacity, cxadj, cadj, nedges, err_line);
}

bm_status bm_mm_info(const char* path, bm_mm_header* header, int64_t* err_line) {
  if (!header) return hfail(BM_ERR_INVALID_ARG, "null header");
  Mapped m;
  if (bm_status s = m.open_file(path)) return s;
  return bm_mm_parse_info(m.p, m.n, header, err_line);
}

bm_status bm_mm_load(const char* path, int32_t threads, int64_t capacity, int64_t* cxadj, int32_t* cadj,
                     int64_t* nedges, int64_t* err_line) {
  Mapped m;
  if (bm_status s = m.open_file(path)) return s;
  return parse_mm(m.p, m.n, threads, capacity, cxadj, cadj, nedges, err_line);
}

bm_status bm_mm_write(const char* path, int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj,
                      int32_t threads) {
  if (!path || nc < 0 || nr < 0 || !cxadj || (cxadj[nc] > 0 && !cadj)) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  threads = resolve_threads(threads);
  FILE* f = std::fopen(path, "wb");
  if (!f) return io_fail(std::string("cannot open '") + path + "' for writing");
  // write_matrix_market (matrix_market.cpp:111-118), byte for byte.
  std::string head = "%%MatrixMarket matrix coordinate pattern general\n";
  char num[96];
  char* o = num;
  o = put_u64(o, (unsigned long long)nr);
  *o++ = ' ';
  o = put_u64(o, (unsigned long long)nc);
  *o++ = ' ';
  o = put_u64(o, (unsigned long long)cxadj[nc]);
  *o++ = '\n';
  head.append(num, o);
  bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
  // Edge-balanced column blocks of about 4M entries, formatted in parallel in
  // batches and written in order.
  std::vector<int32_t> cuts{0};
  const int64_t per = 4LL << 20;
  while (cuts.back() < nc) {
    const int64_t goal = cxadj[cuts.back()] + per;
    int32_t c = (int32_t)(std::upper_bound(cxadj + cuts.back() + 1, cxadj + nc + 1, goal) - cxadj) - 1;
    cuts.push_back(std::max(c, cuts.back() + 1));
  }
  const long long nblk = (long long)cuts.size() - 1, batch = 2LL * threads;
  std::vector<std::string> out((size_t)batch);
  for (long long b0 = 0; b0 < nblk && ok; b0 += batch) {
    const long long nb = std::min(batch, nblk - b0);
    parallel_chunks(nb, threads, [&](long long k) {
      const int32_t c0 = cuts[b0 + k], c1 = cuts[b0 + k + 1];
      std::string& s = out[k];
      s.resize((size_t)(cxadj[c1] - cxadj[c0]) * 24);
      char* w = s.data();
      for (int32_t c = c0; c < c1; ++c)
        for (int64_t j = cxadj[c]; j < cxadj[c + 1]; ++j) {
          w = put_u64(w, (unsigned long long)cadj[j] + 1);
          *w++ = ' ';
          w = put_u64(w, (unsigned long long)c + 1);
          *w++ = '\n';
        }
      s.resize((size_t)(w - s.data()));
    });
    for (long long k = 0; k < nb && ok; ++k) ok = std::fwrite(out[k].data(), 1, out[k].size(), f) == out[k].size();
  }
  ok = (std::fclose(f) == 0) && ok;
  return ok ? BM_OK : io_fail(std::string("write to '") + path + "' failed");
}

bm_status bm_csc_write(const char* path, int32_t nc, int32_t nr, const int64_t* cxadj, const int32_t* cadj,
                       int32_t threads) {
  if (!path || nc < 0 || nr < 0 || !cxadj || (cxadj[nc] > 0 && !cadj)) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  threads = resolve_threads(threads);
  CscHeader h{};
  std::memcpy(h.magic, kMagic, 8);
  h.nc = nc;
  h.nr = nr;
  h.nedges = cxadj[nc];
  h.checksum = csc_checksum(nc, nr, cxadj, cadj, h.nedges, threads);
  const int fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return io_fail(std::string("cannot open '") + path + "' for writing");
  const int64_t off_adj = (int64_t)sizeof h + 8 * ((int64_t)nc + 1);
  bm_status s = pio(fd, true, reinterpret_cast<char*>(&h), sizeof h, 0, 1);
  if (!s) s = pio(fd, true, reinterpret_cast<char*>(const_cast<int64_t*>(cxadj)), 8 * ((int64_t)nc + 1), sizeof h, threads);
  if (!s) s = pio(fd, true, reinterpret_cast<char*>(const_cast<int32_t*>(cadj)), 4 * h.nedges, off_adj, threads);
  if (close(fd) != 0 && !s) s = io_fail(std::string("close of '") + path + "' failed");
  return s;
}

bm_status bm_csc_info(const char* path, int32_t* nc, int32_t* nr, int64_t* nedges) {
  if (!path || !nc || !nr || !nedges) return hfail(BM_ERR_INVALID_ARG, "bad arguments");
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) return io_fail(std::string("cannot open '") + path + "'");
  CscHeader h{};
  struct stat st;
  const bool got = pread(fd, &h, sizeof h, 0) == (ssize_t)sizeof h && fstat(fd, &st) == 0;
  close(fd);
  if (!got || std::memcmp(h.magic, kMagic, 8) != 0) return hfail(BM_ERR_INVALID_ARG, "not a BMCSC001 file");
  if (h.nc < 0 || h.nr < 0 || h.nedges < 0 ||
      (int64_t)st.st_size != (int64_t)sizeof h + 8 * ((int64_t)h.nc + 1) + 4 * h.nedges)
    return hfail(BM_ERR_INVALID_ARG, "BMCSC001 header does not match the file size");
  *nc = h.nc;
  *nr = h.nr;
  *nedges = h.nedges;
  return BM_OK;
}

bm_status bm_csc_read(const char* path, int32_t threads, int64_t capacity, int64_t* cxadj, int32_t* cadj) {
  int32_t nc = 0, nr = 0;
  int64_t ne = 0;
  if (bm_status s = bm_csc_info(path, &nc, &nr, &ne)) return s;
  if (!cxadj || (ne > 0 && !cadj)) return hfail(BM_ERR_INVALID_ARG, "null output buffer");
  if (capacity < ne) return hfail(BM_ERR_INVALID_ARG, "capacity below the file's edge count");
  threads = resolve_threads(threads);
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) return io_fail(std::string("cannot open '") + path + "'");
  CscHeader h{};
  bm_status s = pio(fd, false, reinterpret_cast<char*>(&h), sizeof h, 0, 1);
  if (!s) s = pio(fd, false, reinterpret_cast<char*>(cxadj), 8 * ((int64_t)nc + 1), sizeof h, threads);
  if (!s) s = pio(fd, false, reinterpret_cast<char*>(cadj), 4 * ne, (int64_t)sizeof h + 8 * ((int64_t)nc + 1), threads);
  close(fd);
  if (s) return s;
  if (csc_checksum(nc, nr, cxadj, cadj, ne, threads) != h.checksum)
    return hfail(BM_ERR_INVALID_ARG, "BMCSC001 checksum mismatch (corrupt file)");
  if (cxadj[nc] != ne) return hfail(BM_ERR_INVALID_ARG, "cxadj[nc] does not match the edge count");
  return check_csc_mt(nc, nr, cxadj, cadj, threads);
}

}  // extern "C"
