// qfb_formats.cpp — the reference's on-disk formats, host side (SURVEY.md
// §8 f4), so reference-produced golden tensors and reference-trained scales
// feed the GPU path and our outputs go back to the reference tools:
//
//  - QSIM tensors (tensor_io.hpp:1-125): "QSIM", u32 version = 1, u32 rank,
//    u64 dims[rank], u8 precision tag, little-endian float32 data. Several
//    tensors may follow each other in one blob (checkpoints); parse takes
//    and advances an offset like parse_tensor (tensor_io.hpp:68-99).
//  - QSCL scales (distill.hpp:287-362): "QSCL", u32 version = 1, u64
//    manifest length, a JSON manifest {"version":1,"layers":{name:
//    {"log_w_off","log_w_count","log_a_off"}}} and a float32 payload of the
//    log scales. The writer emits byte-identical files to
//    serialize_scales (layers in name order, compact JSON, integers); the
//    reader accepts any JSON the reference's reader accepts for this schema.
//
// Error behaviour mirrors the reference: every malformed input is
// QFB_ERR_IO with the reference's message (IoError, errors.hpp:21).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/qfb.h"
#include "qfb_kernels.h"

namespace {

using qfb::set_error;

// ------------------------------------------------------------ bytes ---
// Both formats are little-endian on disk. The host is little-endian (x86-64,
// aarch64), so scalars are copied as raw bytes; the static_assert keeps a
// big-endian port from silently writing the wrong byte order.
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "qfb formats assume a little-endian host");

template <typename T>
void put_le(std::string& out, T v) {
  static_assert(std::is_trivially_copyable<T>::value, "raw scalar");
  char raw[sizeof(T)];
  std::memcpy(raw, &v, sizeof(T));
  out.append(raw, sizeof(T));
}

template <typename T>
T get_le(const char* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}

// float32 payloads move by bit pattern (NaN payloads and -0 preserved)
void put_f32(std::string& out, float f) { put_le<float>(out, f); }
float get_f32(const char* p) { return get_le<float>(p); }

bool read_file(const char* path, std::string& out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  out.clear();
  char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) out.append(buf, got);
  const bool ok = !std::ferror(f);
  std::fclose(f);
  return ok;
}

// IoError texts as the reference's writer reports them (tensor_io.hpp:101-106)
qfb_status write_file(const char* path, const std::string& bytes) {
  FILE* f = std::fopen(path, "wb");
  if (!f) return set_error(QFB_ERR_IO, (std::string("cannot open for writing: ") + path).c_str());
  const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
  const bool closed = std::fclose(f) == 0;
  if (!ok || !closed) return set_error(QFB_ERR_IO, (std::string("write failed: ") + path).c_str());
  return QFB_OK;
}

constexpr uint32_t kTensorVersion = 1;  // tensor_io.hpp:53
constexpr uint32_t kScalesVersion = 1;  // distill.hpp:294

// ------------------------------------------------------------- JSON ---
// Minimal JSON reader for the QSCL manifest: objects, arrays, strings with
// escapes, numbers, true/false/null. Numbers keep their text so integer
// offsets are read exactly.
struct JVal {
  enum Kind { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
  std::string text;  // number text or string value
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;

  const JVal* get(const char* key) const {
    const JVal* hit = nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) hit = &kv.second;  // last duplicate wins
    return hit;
  }
};

struct JParser {
  const char* p;
  const char* e;
  std::string err;

  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool fail(const char* m) {
    if (err.empty()) err = m;
    return false;
  }
  bool lit(const char* s) {
    const size_t n = std::strlen(s);
    if ((size_t)(e - p) < n || std::memcmp(p, s, n) != 0) return fail("invalid literal");
    p += n;
    return true;
  }
  static void utf8(std::string& o, uint32_t cp) {
    if (cp < 0x80) {
      o.push_back((char)cp);
    } else if (cp < 0x800) {
      o.push_back((char)(0xc0 | (cp >> 6)));
      o.push_back((char)(0x80 | (cp & 0x3f)));
    } else if (cp < 0x10000) {
      o.push_back((char)(0xe0 | (cp >> 12)));
      o.push_back((char)(0x80 | ((cp >> 6) & 0x3f)));
      o.push_back((char)(0x80 | (cp & 0x3f)));
    } else {
      o.push_back((char)(0xf0 | (cp >> 18)));
      o.push_back((char)(0x80 | ((cp >> 12) & 0x3f)));
      o.push_back((char)(0x80 | ((cp >> 6) & 0x3f)));
      o.push_back((char)(0x80 | (cp & 0x3f)));
    }
  }
  bool hex4(uint32_t& v) {
    if (e - p < 4) return fail("truncated \\u escape");
    v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
      else return fail("bad \\u escape");
    }
    return true;
  }
  bool str(std::string& o) {
    if (p >= e || *p != '"') return fail("expected string");
    ++p;
    while (p < e && *p != '"') {
      const unsigned char c = (unsigned char)*p;
      if (c < 0x20) return fail("control character in string");
      if (c != '\\') {
        o.push_back((char)c);
        ++p;
        continue;
      }
      if (++p >= e) return fail("truncated escape");
      const char x = *p++;
      switch (x) {
        case '"': o.push_back('"'); break;
        case '\\': o.push_back('\\'); break;
        case '/': o.push_back('/'); break;
        case 'b': o.push_back('\b'); break;
        case 'f': o.push_back('\f'); break;
        case 'n': o.push_back('\n'); break;
        case 'r': o.push_back('\r'); break;
        case 't': o.push_back('\t'); break;
        case 'u': {
          uint32_t cp;
          if (!hex4(cp)) return false;
          if (cp >= 0xd800 && cp < 0xdc00) {
            uint32_t lo;
            if (e - p < 2 || p[0] != '\\' || p[1] != 'u') return fail("unpaired surrogate");
            p += 2;
            if (!hex4(lo) || lo < 0xdc00 || lo > 0xdfff) return fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xd800) << 10) + (lo - 0xdc00);
          } else if (cp >= 0xdc00 && cp < 0xe000) {
            return fail("unpaired surrogate");
          }
          utf8(o, cp);
          break;
        }
        default: return fail("bad escape");
      }
    }
    if (p >= e) return fail("unterminated string");
    ++p;
    return true;
  }
  bool num(std::string& o) {
    const char* s = p;
    if (p < e && *p == '-') ++p;
    if (p >= e || !(*p >= '0' && *p <= '9')) return fail("bad number");
    if (*p == '0') ++p;
    else while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p < e && *p == '.') {
      ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) return fail("bad number");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) return fail("bad number");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    o.assign(s, p);
    return true;
  }
  bool value(JVal& v, int depth) {
    if (depth > 64) return fail("nesting too deep");
    ws();
    if (p >= e) return fail("unexpected end of input");
    switch (*p) {
      case '{': {
        ++p;
        v.kind = JVal::kObj;
        ws();
        if (p < e && *p == '}') {
          ++p;
          return true;
        }
        for (;;) {
          ws();
          std::string k;
          if (!str(k)) return false;
          ws();
          if (p >= e || *p != ':') return fail("expected ':'");
          ++p;
          JVal c;
          if (!value(c, depth + 1)) return false;
          v.obj.emplace_back(std::move(k), std::move(c));
          ws();
          if (p < e && *p == ',') {
            ++p;
            continue;
          }
          if (p < e && *p == '}') {
            ++p;
            return true;
          }
          return fail("expected ',' or '}'");
        }
      }
      case '[': {
        ++p;
        v.kind = JVal::kArr;
        ws();
        if (p < e && *p == ']') {
          ++p;
          return true;
        }
        for (;;) {
          JVal c;
          if (!value(c, depth + 1)) return false;
          v.arr.push_back(std::move(c));
          ws();
          if (p < e && *p == ',') {
            ++p;
            continue;
          }
          if (p < e && *p == ']') {
            ++p;
            return true;
          }
          return fail("expected ',' or ']'");
        }
      }
      case '"': v.kind = JVal::kStr; return str(v.text);
      case 't': v.kind = JVal::kBool; v.text = "true"; return lit("true");
      case 'f': v.kind = JVal::kBool; v.text = "false"; return lit("false");
      case 'n': v.kind = JVal::kNull; return lit("null");
      default: v.kind = JVal::kNum; return num(v.text);
    }
  }
  bool document(JVal& v) {
    if (!value(v, 0)) return false;
    ws();
    if (p != e) return fail("trailing characters");
    return true;
  }
};

// Unsigned integer of a manifest field (nlohmann get<size_t>: numbers that
// are non-negative integers; anything else is a type error).
bool as_size(const JVal* v, uint64_t& out) {
  if (!v || v->kind != JVal::kNum) return false;
  const std::string& t = v->text;
  if (t.empty() || t[0] == '-' || t.find_first_of(".eE") != std::string::npos) return false;
  uint64_t r = 0;
  for (char c : t) {
    const uint64_t d = (uint64_t)(c - '0');
    if (r > (UINT64_MAX - d) / 10) return false;
    r = r * 10 + d;
  }
  out = r;
  return true;
}

// nlohmann::json::dump() string escaping (ASCII control characters as
// \uXXXX except the short forms; everything else byte-for-byte).
void json_escape(std::string& o, const std::string& s) {
  o.push_back('"');
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", c);
          o += buf;
        } else {
          o.push_back((char)c);
        }
    }
  }
  o.push_back('"');
}

}  // namespace

struct qfb_tensor_file {
  std::vector<int64_t> shape;
  uint8_t precision = 0;
  std::vector<float> data;
};

struct qfb_scales {
  std::map<std::string, std::pair<std::vector<double>, double>> by_layer;  // sorted like ScaleSet
  std::vector<std::string> names;                                          // by_layer order
};

extern "C" {

// ------------------------------------------------------------- QSIM ---
qfb_status qfb_qsim_parse(const void* buf, size_t size, size_t* offset, qfb_tensor_file** out) {
  if (!buf || !offset || !out) return set_error(QFB_ERR_VALUE, "qsim_parse: null argument");
  *out = nullptr;
  const char* b = static_cast<const char*>(buf);
  size_t off = *offset;
  auto need = [&](size_t n) { return off <= size && n <= size - off; };
  if (!need(12)) return set_error(QFB_ERR_IO, "tensor blob truncated");
  if (std::memcmp(b + off, "QSIM", 4) != 0) return set_error(QFB_ERR_IO, "bad tensor magic (expected QSIM)");
  const uint32_t ver = get_le<uint32_t>(b + off + 4);
  if (ver != kTensorVersion)
    return set_error(QFB_ERR_IO, ("unsupported tensor format version " + std::to_string(ver)).c_str());
  const uint32_t rank = get_le<uint32_t>(b + off + 8);
  off += 12;
  if ((uint64_t)rank > (size - std::min(off, size)) / 8 || !need(8 * (size_t)rank + 1))
    return set_error(QFB_ERR_IO, "tensor blob truncated");
  qfb_tensor_file* t = new qfb_tensor_file();
  uint64_t n = 1;
  bool overflow = false, nonpos = false;
  for (uint32_t i = 0; i < rank; ++i) {
    const uint64_t d = get_le<uint64_t>(b + off);
    off += 8;
    t->shape.push_back((int64_t)d);
    if ((int64_t)d <= 0) nonpos = true;
    else if (n > UINT64_MAX / d) overflow = true;
    else n *= d;
  }
  if (nonpos) {  // the Tensor constructor rejects it (tensor.hpp:66-73)
    delete t;
    return set_error(QFB_ERR_SHAPE, "non-positive dim in tensor shape");
  }
  t->precision = static_cast<uint8_t>(b[off]);
  off += 1;
  if (overflow || n > (size - off) / 4) {
    delete t;
    return set_error(QFB_ERR_IO, "tensor blob truncated");
  }
  t->data.resize((size_t)n);
  for (uint64_t i = 0; i < n; ++i) t->data[(size_t)i] = get_f32(b + off + 4 * i);
  off += 4 * (size_t)n;
  *offset = off;
  *out = t;
  return QFB_OK;
}

qfb_status qfb_qsim_load(const char* path, qfb_tensor_file** out) {
  if (!path || !out) return set_error(QFB_ERR_VALUE, "qsim_load: null argument");
  *out = nullptr;
  std::string buf;
  if (!read_file(path, buf)) return set_error(QFB_ERR_IO, (std::string("cannot open: ") + path).c_str());
  size_t off = 0;
  if (qfb_status st = qfb_qsim_parse(buf.data(), buf.size(), &off, out)) return st;
  if (off != buf.size()) {
    qfb_qsim_free(*out);
    *out = nullptr;
    return set_error(QFB_ERR_IO, (std::string("trailing bytes in tensor file ") + path).c_str());
  }
  return QFB_OK;
}

qfb_status qfb_qsim_info(const qfb_tensor_file* t, int32_t* rank, const int64_t** shape,
                         int32_t* precision, int64_t* numel, const float** data) {
  if (!t) return set_error(QFB_ERR_VALUE, "qsim_info: null tensor");
  if (rank) *rank = (int32_t)t->shape.size();
  if (shape) *shape = t->shape.data();
  if (precision) *precision = t->precision;
  if (numel) *numel = (int64_t)t->data.size();
  if (data) *data = t->data.data();
  return QFB_OK;
}

void qfb_qsim_free(qfb_tensor_file* t) { delete t; }

qfb_status qfb_qsim_serialize(const float* data, int32_t rank, const int64_t* shape,
                              int32_t precision, char* out, size_t cap, size_t* size) {
  if (rank < 0 || (rank > 0 && !shape) || !size) return set_error(QFB_ERR_VALUE, "qsim_serialize: bad arguments");
  uint64_t n = 1;
  for (int32_t i = 0; i < rank; ++i) {
    if (shape[i] <= 0) return set_error(QFB_ERR_SHAPE, "non-positive dim in tensor shape");  // tensor.hpp:69
    n *= (uint64_t)shape[i];
  }
  if (n > 0 && !data) return set_error(QFB_ERR_VALUE, "qsim_serialize: null data");
  const size_t need = 13 + 8 * (size_t)rank + 4 * (size_t)n;  // magic, version, rank, tag
  *size = need;
  if (!out) return QFB_OK;  // size query
  if (cap < need) return set_error(QFB_ERR_VALUE, "qsim_serialize: buffer too small");
  std::string s;
  s.reserve(need);
  s.append("QSIM", 4);
  put_le<uint32_t>(s, kTensorVersion);
  put_le<uint32_t>(s, (uint32_t)rank);
  for (int32_t i = 0; i < rank; ++i) put_le<uint64_t>(s, (uint64_t)shape[i]);
  s.push_back(static_cast<char>(static_cast<uint8_t>(precision)));
  for (uint64_t i = 0; i < n; ++i) put_f32(s, data[i]);
  std::memcpy(out, s.data(), need);
  return QFB_OK;
}

qfb_status qfb_qsim_save(const char* path, const float* data, int32_t rank, const int64_t* shape,
                         int32_t precision) {
  if (!path) return set_error(QFB_ERR_VALUE, "qsim_save: null path");
  size_t need = 0;
  if (qfb_status st = qfb_qsim_serialize(data, rank, shape, precision, nullptr, 0, &need)) return st;
  std::string s(need, '\0');
  if (qfb_status st = qfb_qsim_serialize(data, rank, shape, precision, &s[0], need, &need)) return st;
  return write_file(path, s);
}

// ------------------------------------------------------------- QSCL ---
qfb_status qfb_qscl_parse(const void* buf, size_t size, qfb_scales** out) {
  if (!buf || !out) return set_error(QFB_ERR_VALUE, "qscl_parse: null argument");
  *out = nullptr;
  const char* b = static_cast<const char*>(buf);
  if (size < 16 || std::memcmp(b, "QSCL", 4) != 0) return set_error(QFB_ERR_IO, "bad scales magic (expected QSCL)");
  const uint32_t ver = get_le<uint32_t>(b + 4);
  if (ver != kScalesVersion)
    return set_error(QFB_ERR_IO, ("unsupported scales version " + std::to_string(ver)).c_str());
  const uint64_t mlen = get_le<uint64_t>(b + 8);
  if (mlen > size - 16) return set_error(QFB_ERR_IO, "scales manifest out of bounds");
  JParser jp{b + 16, b + 16 + mlen, {}};
  JVal man;
  if (!jp.document(man)) return set_error(QFB_ERR_IO, ("scales manifest parse error: " + jp.err).c_str());
  const JVal* layers = man.kind == JVal::kObj ? man.get("layers") : nullptr;
  if (!layers || layers->kind != JVal::kObj)
    return set_error(QFB_ERR_IO, "scales manifest: missing or invalid 'layers' object");
  const size_t base = 16 + (size_t)mlen;
  qfb_scales* set = new qfb_scales();
  for (const auto& kv : layers->obj) {
    uint64_t woff = 0, wcount = 0, aoff = 0;
    const JVal& jl = kv.second;
    if (jl.kind != JVal::kObj || !as_size(jl.get("log_w_off"), woff) ||
        !as_size(jl.get("log_w_count"), wcount) || !as_size(jl.get("log_a_off"), aoff)) {
      delete set;
      return set_error(QFB_ERR_IO, ("scales manifest: bad entry for layer '" + kv.first + "'").c_str());
    }
    // distill.hpp:340-343 bounds check (overflow-safe form)
    const uint64_t sz = size;
    if (woff > sz || aoff > sz || base > sz - woff || wcount > (sz - woff - base) / 4 ||
        base > sz - aoff || 4 > sz - aoff - base) {
      delete set;
      return set_error(QFB_ERR_IO, "scales payload truncated");
    }
    std::vector<double> w((size_t)wcount);
    for (uint64_t i = 0; i < wcount; ++i) w[(size_t)i] = (double)get_f32(b + base + woff + 4 * i);
    const double a = (double)get_f32(b + base + aoff);
    set->by_layer[kv.first] = {std::move(w), a};  // duplicate keys: the last wins
  }
  for (const auto& kv : set->by_layer) set->names.push_back(kv.first);
  *out = set;
  return QFB_OK;
}

qfb_status qfb_qscl_load(const char* path, qfb_scales** out) {
  if (!path || !out) return set_error(QFB_ERR_VALUE, "qscl_load: null argument");
  *out = nullptr;
  std::string buf;
  if (!read_file(path, buf)) return set_error(QFB_ERR_IO, (std::string("cannot open: ") + path).c_str());
  return qfb_qscl_parse(buf.data(), buf.size(), out);
}

int32_t qfb_qscl_count(const qfb_scales* s) { return s ? (int32_t)s->names.size() : 0; }

qfb_status qfb_qscl_layer(const qfb_scales* s, int32_t i, const char** name, const double** log_w,
                          int64_t* count, double* log_a) {
  if (!s || i < 0 || i >= (int32_t)s->names.size()) return set_error(QFB_ERR_VALUE, "qscl_layer: index out of range");
  const auto& e = s->by_layer.at(s->names[(size_t)i]);
  if (name) *name = s->names[(size_t)i].c_str();
  if (log_w) *log_w = e.first.data();
  if (count) *count = (int64_t)e.first.size();
  if (log_a) *log_a = e.second;
  return QFB_OK;
}

void qfb_qscl_free(qfb_scales* s) { delete s; }

qfb_status qfb_qscl_serialize(int32_t n, const char* const* names, const double* const* log_w,
                              const int64_t* counts, const double* log_a, char* out, size_t cap,
                              size_t* size) {
  if (n < 0 || !size || (n > 0 && (!names || !log_w || !counts || !log_a)))
    return set_error(QFB_ERR_VALUE, "qscl_serialize: bad arguments");
  // ScaleSet::by_layer is a std::map: layers in name order, unique names
  std::map<std::string, int32_t> order;
  for (int32_t i = 0; i < n; ++i) {
    if (!names[i] || counts[i] < 0 || (counts[i] > 0 && !log_w[i]))
      return set_error(QFB_ERR_VALUE, "qscl_serialize: bad layer entry");
    order[names[i]] = i;  // a repeated name keeps the last entry, like map assignment
  }
  std::string payload, man = "{\"version\":" + std::to_string(kScalesVersion) + ",\"layers\":{";
  bool first = true;
  for (const auto& kv : order) {
    const int32_t i = kv.second;
    if (!first) man.push_back(',');
    first = false;
    json_escape(man, kv.first);
    man += ":{\"log_w_off\":" + std::to_string(payload.size());
    man += ",\"log_w_count\":" + std::to_string(counts[i]);
    for (int64_t k = 0; k < counts[i]; ++k) put_f32(payload, (float)log_w[i][k]);
    man += ",\"log_a_off\":" + std::to_string(payload.size()) + "}";
    put_f32(payload, (float)log_a[i]);
  }
  man += "}}";
  std::string s;
  s.append("QSCL", 4);
  put_le<uint32_t>(s, kScalesVersion);
  put_le<uint64_t>(s, (uint64_t)man.size());
  s += man;
  s += payload;
  *size = s.size();
  if (!out) return QFB_OK;
  if (cap < s.size()) return set_error(QFB_ERR_VALUE, "qscl_serialize: buffer too small");
  std::memcpy(out, s.data(), s.size());
  return QFB_OK;
}

qfb_status qfb_qscl_save(const char* path, int32_t n, const char* const* names, const double* const* log_w,
                         const int64_t* counts, const double* log_a) {
  if (!path) return set_error(QFB_ERR_VALUE, "qscl_save: null path");
  size_t need = 0;
  if (qfb_status st = qfb_qscl_serialize(n, names, log_w, counts, log_a, nullptr, 0, &need)) return st;
  std::string s(need, '\0');
  if (qfb_status st = qfb_qscl_serialize(n, names, log_w, counts, log_a, &s[0], need, &need)) return st;
  return write_file(path, s);
}

}  // extern "C"
