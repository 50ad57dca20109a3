// xs_ingest.cu -- native decoder of XSTRACE1 trace chunks into columns.
//
// Replaces the per-record Python loop of traceio._decode_chunk
// (traceio.py:214-240; layout docs/trace-format.md:20-50): 7.99 s per 1M
// events in the reference.  Host code on purpose: a
// chunk is a stream of length-prefixed 46/54-byte records whose boundaries
// are only known by walking the length prefixes, and decoding on the host
// writes 37 bytes per event of columns (which the device upload then moves
// once) instead of shipping ~50 raw bytes per record plus offsets.  Chunks
// are independent: the Python caller decodes them on a thread pool (ctypes
// releases the GIL), writing straight into the final column arrays.
//
// Error behaviour mirrors traceio: a short buffer anywhere is "truncated at
// byte N", a bad magic / version / category / string index / correlation
// flag is reported with the reference's wording; the caller raises
// TraceFormatError(message).
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "xstrace_b200.h"

namespace {

constexpr char kMagic[8] = {'X', 'S', 'T', 'R', 'A', 'C', 'E', '1'};
constexpr int kVersion = 1;
constexpr int kHeader = 26;

struct Cur {
  const uint8_t* b;
  int64_t n, pos;
  char* err;
  int errlen;
  const char* ctx;
  bool fail(const char* msg) {
    if (err && errlen > 0) snprintf(err, errlen, "%s", msg);
    return false;
  }
  bool need(int64_t k) {
    if (pos + k > n) {
      if (err && errlen > 0) snprintf(err, errlen, "format error: %s truncated at byte %lld", ctx, (long long)pos);
      return false;
    }
    return true;
  }
  template <class T>
  T rd(int64_t at) const {
    T v;
    memcpy(&v, b + at, sizeof(T));
    return v;
  }
};

}  // namespace

extern "C" {

// Header + string table; str_off/str_len (n_strings each) may be null on the
// first call (sizes only).
int xs_chunk_info(const uint8_t* buf, int64_t len, const char* context, xs_chunk_info_t* info, int64_t* str_off,
                  int64_t* str_len, char* err, int errlen) {
  Cur c{buf, len, 0, err, errlen, context ? context : "chunk"};
  if (!c.need(kHeader)) return 1;
  if (memcmp(buf, kMagic, 8) != 0) {
    char m[160];
    snprintf(m, sizeof m, "format error: bad magic in %s", c.ctx);
    c.fail(m);
    return 2;  // the caller formats the reference's repr of the magic
  }
  info->version = c.rd<uint16_t>(8);
  info->clock_domain = (int64_t)c.rd<uint64_t>(10);
  info->chunk_index = (int32_t)c.rd<uint32_t>(18);
  info->n_records = (int32_t)c.rd<uint32_t>(22);
  if (info->version != kVersion) {
    char m[160];
    snprintf(m, sizeof m, "format error: unsupported version %d in %s", info->version, c.ctx);
    c.fail(m);
    return 3;
  }
  c.pos = kHeader;
  if (!c.need(4)) return 1;
  const uint32_t ns = c.rd<uint32_t>(c.pos);
  c.pos += 4;
  info->n_strings = (int32_t)ns;
  for (uint32_t i = 0; i < ns; i++) {
    if (!c.need(4)) return 1;
    const uint32_t l = c.rd<uint32_t>(c.pos);
    c.pos += 4;
    if (!c.need(l)) return 1;
    if (str_off) str_off[i] = c.pos;
    if (str_len) str_len[i] = l;
    c.pos += l;
  }
  info->records_offset = c.pos;
  return 0;
}

// Decode the records of one chunk into the output columns (n_records rows
// each).  name_map maps the chunk's string index to the caller's global
// name rank.  Returns 0, or 1 with the reference-worded message in err.
int xs_chunk_decode(const uint8_t* buf, int64_t len, const char* context, const xs_chunk_info_t* info,
                    const int32_t* name_map, int64_t* pid, int64_t* tid, uint8_t* cat, int32_t* name, int64_t* start,
                    int64_t* dur, int64_t* corr, uint8_t* has_corr, char* err, int errlen) {
  Cur c{buf, len, info->records_offset, err, errlen, context ? context : "chunk"};
  const uint32_t nstr = (uint32_t)info->n_strings;
  for (int32_t r = 0; r < info->n_records; r++) {
    if (!c.need(4)) return 1;
    const uint32_t body = c.rd<uint32_t>(c.pos);
    c.pos += 4;
    if (!c.need(body)) return 1;
    const int64_t b0 = c.pos, end = c.pos + body;
    Cur bc{buf + b0, (int64_t)body, 0, err, errlen, c.ctx};  // the body is its own reader (positions relative)
    if (!bc.need(37)) return 1;
    pid[r] = bc.rd<int64_t>(0);
    tid[r] = bc.rd<int64_t>(8);
    const uint8_t k = bc.b[16];
    const uint32_t ni = bc.rd<uint32_t>(17);
    start[r] = (int64_t)bc.rd<uint64_t>(21);
    dur[r] = (int64_t)bc.rd<uint64_t>(29);
    if (k > 5) {
      char m[160];
      snprintf(m, sizeof m, "format error: unknown category %u in %s", (unsigned)k, c.ctx);
      return c.fail(m), 1;
    }
    if (ni >= nstr) {
      char m[160];
      snprintf(m, sizeof m, "format error: string index %u out of range in %s", ni, c.ctx);
      return c.fail(m), 1;
    }
    cat[r] = k;
    name[r] = name_map[ni];
    bc.pos = 37;
    if (!bc.need(1)) return 1;
    const uint8_t f = bc.b[37];
    if (f == 1) {
      bc.pos = 38;
      if (!bc.need(8)) return 1;
      corr[r] = bc.rd<int64_t>(38);
      has_corr[r] = 1;
    } else if (f == 0) {
      corr[r] = 0;
      has_corr[r] = 0;
    } else {
      char m[160];
      snprintf(m, sizeof m, "format error: bad correlation flag %u in %s", (unsigned)f, c.ctx);
      return c.fail(m), 1;
    }
    c.pos = end;
  }
  return 0;
}

}  // extern "C"
