// DZDL container parsing and payload inflation — the host side of the delta swap-in path
// (formats.read_delta, formats.py:102-169; lossless_decode, compress.py:560-564).
//
// The parser walks the container in place (the caller mmaps the file) and returns per-layer
// byte ranges, so the reference-layout payloads can be copied from the page cache into pinned
// staging buffers and on to the GPU without an intermediate Python copy. Error behaviour
// mirrors the reference reader: every truncation reports the byte offset where reading
// failed, a bad magic / version is rejected, and trailing bytes after the last layer are an
// error. The JSON header stays with the caller (it only carries the configuration).
#include <zlib.h>

#include <cstdint>
#include <cstring>

#include "../../include/dz_b200.h"

namespace {

struct Cursor {
  const uint8_t* buf;
  int64_t len, pos;
  int64_t* err_off;
  bool take(int64_t n, int64_t* off) {
    if (n < 0 || pos + n > len) {
      if (err_off) *err_off = pos;
      return false;
    }
    if (off) *off = pos;
    pos += n;
    return true;
  }
  bool u16(uint32_t* v) {
    int64_t o;
    if (!take(2, &o)) return false;
    *v = static_cast<uint32_t>(buf[o]) | (static_cast<uint32_t>(buf[o + 1]) << 8);
    return true;
  }
  bool u32(uint32_t* v) {
    int64_t o;
    if (!take(4, &o)) return false;
    *v = static_cast<uint32_t>(buf[o]) | (static_cast<uint32_t>(buf[o + 1]) << 8) |
         (static_cast<uint32_t>(buf[o + 2]) << 16) | (static_cast<uint32_t>(buf[o + 3]) << 24);
    return true;
  }
};

}  // namespace

extern "C" int dz_dzdl_parse_header(const uint8_t* buf, int64_t len, dz_dzdl_info* info, int64_t* err_offset) {
  if (!buf || !info || len < 0) return DZ_E_VALUE;
  std::memset(info, 0, sizeof(*info));
  Cursor c{buf, len, 0, err_offset};
  int64_t o;
  if (!c.take(4, &o)) return DZ_E_FORMAT;
  if (std::memcmp(buf, "DZDL", 4) != 0) {
    if (err_offset) *err_offset = 0;
    return DZ_E_FORMAT;  // "bad magic"
  }
  uint32_t version, flags, hlen;
  if (!c.u16(&version)) return DZ_E_FORMAT;
  info->version = static_cast<int32_t>(version);
  if (version != 1) {
    if (err_offset) *err_offset = 4;
    return DZ_E_UNSUPPORTED;  // "unsupported version"
  }
  if (!c.u16(&flags) || !c.u32(&hlen)) return DZ_E_FORMAT;
  info->flags = static_cast<int32_t>(flags);
  info->lossless = (flags & 1u) ? 1 : 0;
  if (!c.take(hlen, &o)) return DZ_E_FORMAT;
  info->header_off = o;
  info->header_len = hlen;
  info->layers_off = c.pos;
  return DZ_OK;
}

extern "C" int dz_dzdl_parse_layers(const uint8_t* buf, int64_t len, int64_t layers_off, int32_t layer_count,
                                    dz_dzdl_layer* layers, int64_t* err_offset) {
  if (!buf || (!layers && layer_count > 0) || layer_count < 0 || layers_off < 0) return DZ_E_VALUE;
  Cursor c{buf, len, layers_off, err_offset};
  for (int32_t i = 0; i < layer_count; i++) {
    dz_dzdl_layer& L = layers[i];
    std::memset(&L, 0, sizeof(L));
    uint32_t nlen, rows, cols, slen, ilen, plen;
    if (!c.u16(&nlen) || !c.take(nlen, &L.name_off)) return DZ_E_FORMAT;
    L.name_len = static_cast<int32_t>(nlen);
    if (!c.u32(&rows) || !c.u32(&cols)) return DZ_E_FORMAT;
    L.rows = static_cast<int32_t>(rows);
    L.cols = static_cast<int32_t>(cols);
    if (!c.u32(&slen) || !c.take(slen, &L.scales_off)) return DZ_E_FORMAT;
    L.scales_len = slen;
    if (!c.u32(&ilen) || !c.take(ilen, &L.index_off)) return DZ_E_FORMAT;
    L.index_len = ilen;
    if (!c.u32(&plen) || !c.take(plen, &L.payload_off)) return DZ_E_FORMAT;
    L.payload_len = plen;
  }
  if (c.pos != len) {
    if (err_offset) *err_offset = c.pos;
    return DZ_E_VALUE;  // trailing bytes after the last layer
  }
  return DZ_OK;
}

extern "C" int dz_inflate(const uint8_t* src, int64_t n, uint8_t* dst, int64_t cap, int64_t* out_len) {
  if (!src || n < 0 || !out_len || cap < 0) return DZ_E_VALUE;
  z_stream zs;
  std::memset(&zs, 0, sizeof(zs));
  if (inflateInit(&zs) != Z_OK) return DZ_E_VALUE;
  zs.next_in = const_cast<Bytef*>(src);
  zs.avail_in = static_cast<uInt>(n);
  uint8_t scratch[16384];
  int64_t total = 0;
  int rc = Z_OK;
  while (rc == Z_OK) {
    const bool direct = dst != nullptr && total < cap;
    zs.next_out = direct ? dst + total : scratch;
    const int64_t room = direct ? cap - total : static_cast<int64_t>(sizeof(scratch));
    zs.avail_out = static_cast<uInt>(room > (1 << 30) ? (1 << 30) : room);
    const uInt before = zs.avail_out;
    rc = inflate(&zs, Z_NO_FLUSH);
    total += before - zs.avail_out;
    if (rc == Z_BUF_ERROR && zs.avail_in == 0) break;  // truncated stream
  }
  inflateEnd(&zs);
  *out_len = total;
  if (rc != Z_STREAM_END) return DZ_E_FORMAT;  // "corrupt lossless stream"
  return total <= cap ? DZ_OK : DZ_E_ENCODING;  // dst too small: *out_len = the size needed
}
