// Tokenization pipeline producer, host C++.
//
// The reference (pipeline.py:264-422, tokenizers.py) tokenizes an indexed JSONL
// corpus with a reader thread, W worker *processes* and an order-restoring
// writer. Here: a reader, W worker threads that each take whole batches of
// documents (no Python, no pickling), and the writer restoring batch order, so
// the CFPKD001 output is byte-identical for any W (and to the reference's).
//
// Per document (pipeline.py:_tokenize_batch):
//   extract_text: the bytes must decode (json.detect_encoding + 'surrogatepass')
//     and parse as one JSON object (Python json grammar: NaN / Infinity allowed,
//     control characters in strings rejected, duplicate keys -> last wins, no
//     trailing data) else MALFORMED; the text key must hold a string else
//     MISSING_TEXT.
//   encode: byte (UTF-8 bytes), whitespace (str.split() on Unicode whitespace,
//     vocabulary lookup, unk), or byte-level BPE over the whole document
//     (lowest-rank merge anywhere, ties to the leftmost, until none applies).
//   empty encodings are skipped; eod appended when enabled.
// A string holding a lone surrogate cannot be UTF-8 encoded: the reference's
// byte / bpe tokenizers raise there and the whole run fails -- so does this
// one (B2S_EINVAL with the document ordinal).
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/b2s.h"

namespace b2s {
void set_error(const char* fmt, ...);
}

namespace {

// ------------------------------------------------------------------ code points
// A decoded JSON string: Unicode code points, surrogates (0xD800-0xDFFF) kept
// as lone code points exactly like a Python str built with 'surrogatepass'.
using U32 = std::vector<uint32_t>;

bool is_surrogate(uint32_t c) { return c >= 0xD800 && c <= 0xDFFF; }

// Python str.isspace() for the characters str.split() splits on.
bool py_isspace(uint32_t c) {
  if (c == 0x20 || (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x1F)) return true;
  if (c < 0x85) return false;
  return c == 0x85 || c == 0xA0 || c == 0x1680 || (c >= 0x2000 && c <= 0x200A) || c == 0x2028 ||
         c == 0x2029 || c == 0x202F || c == 0x205F || c == 0x3000;
}

// UTF-8 encode (fails on surrogates, like str.encode('utf-8')).
bool utf8_encode(const uint32_t* p, size_t n, std::string& out) {
  for (size_t i = 0; i < n; ++i) {
    const uint32_t c = p[i];
    if (is_surrogate(c)) return false;
    if (c < 0x80) {
      out.push_back((char)c);
    } else if (c < 0x800) {
      out.push_back((char)(0xC0 | (c >> 6)));
      out.push_back((char)(0x80 | (c & 0x3F)));
    } else if (c < 0x10000) {
      out.push_back((char)(0xE0 | (c >> 12)));
      out.push_back((char)(0x80 | ((c >> 6) & 0x3F)));
      out.push_back((char)(0x80 | (c & 0x3F)));
    } else {
      out.push_back((char)(0xF0 | (c >> 18)));
      out.push_back((char)(0x80 | ((c >> 12) & 0x3F)));
      out.push_back((char)(0x80 | ((c >> 6) & 0x3F)));
      out.push_back((char)(0x80 | (c & 0x3F)));
    }
  }
  return true;
}

// Strict UTF-8 decode with 'surrogatepass' (encoded surrogates ED A0..BF xx accepted).
bool utf8_decode(const uint8_t* s, size_t n, U32& out) {
  size_t i = 0;
  while (i < n) {
    const uint8_t b = s[i];
    uint32_t c;
    int k;
    if (b < 0x80) { out.push_back(b); ++i; continue; }
    if (b >= 0xC2 && b <= 0xDF) { c = b & 0x1F; k = 1; }
    else if (b >= 0xE0 && b <= 0xEF) { c = b & 0x0F; k = 2; }
    else if (b >= 0xF0 && b <= 0xF4) { c = b & 0x07; k = 3; }
    else return false;
    for (int j = 1; j <= k; ++j) {
      if (i + j >= n) return false;
      const uint8_t t = s[i + j];
      if ((t & 0xC0) != 0x80) return false;
      c = (c << 6) | (t & 0x3F);
    }
    if ((k == 2 && c < 0x800) || (k == 3 && (c < 0x10000 || c > 0x10FFFF))) return false;
    out.push_back(c);
    i += k + 1;
  }
  return true;
}

bool utf16_decode(const uint8_t* s, size_t n, bool be, U32& out) {
  if (n % 2) return false;
  for (size_t i = 0; i < n; i += 2) {
    uint32_t u = be ? ((uint32_t)s[i] << 8 | s[i + 1]) : ((uint32_t)s[i + 1] << 8 | s[i]);
    if (u >= 0xD800 && u <= 0xDBFF && i + 3 < n) {
      const uint32_t v = be ? ((uint32_t)s[i + 2] << 8 | s[i + 3]) : ((uint32_t)s[i + 3] << 8 | s[i + 2]);
      if (v >= 0xDC00 && v <= 0xDFFF) {
        out.push_back(0x10000 + ((u - 0xD800) << 10) + (v - 0xDC00));
        i += 2;
        continue;
      }
    }
    out.push_back(u);  // surrogatepass keeps lone surrogates
  }
  return true;
}

bool utf32_decode(const uint8_t* s, size_t n, bool be, U32& out) {
  if (n % 4) return false;
  for (size_t i = 0; i < n; i += 4) {
    const uint32_t c = be ? ((uint32_t)s[i] << 24 | (uint32_t)s[i + 1] << 16 | (uint32_t)s[i + 2] << 8 | s[i + 3])
                          : ((uint32_t)s[i + 3] << 24 | (uint32_t)s[i + 2] << 16 | (uint32_t)s[i + 1] << 8 | s[i]);
    if (c > 0x10FFFF) return false;
    out.push_back(c);
  }
  return true;
}

// json.loads(bytes): detect_encoding, then decode with 'surrogatepass'.
bool decode_json_bytes(const uint8_t* s, size_t n, U32& out) {
  auto starts = [&](const char* pre, size_t k) { return n >= k && memcmp(s, pre, k) == 0; };
  if (starts("\x00\x00\xFE\xFF", 4)) return utf32_decode(s + 4, n - 4, true, out);
  if (starts("\xFF\xFE\x00\x00", 4)) return utf32_decode(s + 4, n - 4, false, out);
  if (starts("\xFE\xFF", 2)) return utf16_decode(s + 2, n - 2, true, out);
  if (starts("\xFF\xFE", 2)) return utf16_decode(s + 2, n - 2, false, out);
  if (starts("\xEF\xBB\xBF", 3)) return utf8_decode(s + 3, n - 3, out);
  if (n >= 4) {
    if (!s[0]) return s[1] ? utf16_decode(s, n, true, out) : utf32_decode(s, n, true, out);
    if (!s[1]) return (s[2] || s[3]) ? utf16_decode(s, n, false, out) : utf32_decode(s, n, false, out);
  } else if (n == 2) {
    if (!s[0]) return utf16_decode(s, n, true, out);
    if (!s[1]) return utf16_decode(s, n, false, out);
  }
  return utf8_decode(s, n, out);
}

// ------------------------------------------------------------------ JSON (Python json grammar)
struct Json {
  const U32& t;
  size_t i = 0;
  explicit Json(const U32& text) : t(text) {}
  void ws() {
    while (i < t.size() && (t[i] == ' ' || t[i] == '\t' || t[i] == '\n' || t[i] == '\r')) ++i;
  }
  bool lit(const char* w) {
    size_t k = 0;
    for (; w[k]; ++k)
      if (i + k >= t.size() || t[i + k] != (uint32_t)(unsigned char)w[k]) return false;
    i += k;
    return true;
  }
  static int hex(uint32_t c) {
    if (c >= '0' && c <= '9') return (int)(c - '0');
    if (c >= 'a' && c <= 'f') return (int)(c - 'a' + 10);
    if (c >= 'A' && c <= 'F') return (int)(c - 'A' + 10);
    return -1;
  }
  bool u4(uint32_t& v) {
    if (i + 4 > t.size()) return false;
    v = 0;
    for (int k = 0; k < 4; ++k) {
      const int h = hex(t[i + k]);
      if (h < 0) return false;
      v = v * 16 + (uint32_t)h;
    }
    i += 4;
    return true;
  }
  // at the opening quote; decoded string into out (or skipped when out == nullptr)
  bool string(U32* out) {
    ++i;
    while (true) {
      if (i >= t.size()) return false;
      const uint32_t c = t[i];
      if (c == '"') { ++i; return true; }
      if (c < 0x20) return false;  // strict: control characters not allowed
      if (c != '\\') { if (out) out->push_back(c); ++i; continue; }
      ++i;
      if (i >= t.size()) return false;
      const uint32_t e = t[i++];
      uint32_t v;
      switch (e) {
        case '"': v = '"'; break;
        case '\\': v = '\\'; break;
        case '/': v = '/'; break;
        case 'b': v = 8; break;
        case 'f': v = 12; break;
        case 'n': v = 10; break;
        case 'r': v = 13; break;
        case 't': v = 9; break;
        case 'u': {
          if (!u4(v)) return false;
          if (v >= 0xD800 && v <= 0xDBFF && i + 1 < t.size() && t[i] == '\\' && t[i + 1] == 'u') {
            const size_t save = i;
            i += 2;
            uint32_t w;
            if (u4(w) && w >= 0xDC00 && w <= 0xDFFF) v = 0x10000 + ((v - 0xD800) << 10) + (w - 0xDC00);
            else i = save;  // the second escape is parsed on its own (lone surrogate kept)
          }
          break;
        }
        default: return false;
      }
      if (out) out->push_back(v);
    }
  }
  bool number() {  // -?(0|[1-9]\d*)(\.\d+)?([eE][-+]?\d+)?  or -Infinity
    if (i < t.size() && t[i] == '-') {
      ++i;
      if (lit("Infinity")) return true;
    }
    auto digit = [&](size_t k) { return k < t.size() && t[k] >= '0' && t[k] <= '9'; };
    if (!digit(i)) return false;
    if (t[i] == '0') ++i;
    else while (digit(i)) ++i;
    if (i < t.size() && t[i] == '.' && digit(i + 1)) { ++i; while (digit(i)) ++i; }
    if (i < t.size() && (t[i] == 'e' || t[i] == 'E')) {
      size_t k = i + 1;
      if (k < t.size() && (t[k] == '+' || t[k] == '-')) ++k;
      if (digit(k)) { i = k; while (digit(i)) ++i; }
    }
    return true;
  }
  // any value (iterative over nesting); strings skipped
  bool value(int depth = 0) {
    if (depth > 100000) return false;
    ws();
    if (i >= t.size()) return false;
    const uint32_t c = t[i];
    if (c == '"') return string(nullptr);
    if (c == '{') {
      ++i; ws();
      if (i < t.size() && t[i] == '}') { ++i; return true; }
      while (true) {
        ws();
        if (i >= t.size() || t[i] != '"' || !string(nullptr)) return false;
        ws();
        if (i >= t.size() || t[i] != ':') return false;
        ++i;
        if (!value(depth + 1)) return false;
        ws();
        if (i < t.size() && t[i] == ',') { ++i; continue; }
        if (i < t.size() && t[i] == '}') { ++i; return true; }
        return false;
      }
    }
    if (c == '[') {
      ++i; ws();
      if (i < t.size() && t[i] == ']') { ++i; return true; }
      while (true) {
        if (!value(depth + 1)) return false;
        ws();
        if (i < t.size() && t[i] == ',') { ++i; continue; }
        if (i < t.size() && t[i] == ']') { ++i; return true; }
        return false;
      }
    }
    if (lit("null") || lit("true") || lit("false") || lit("NaN") || lit("Infinity")) return true;
    return number();
  }
};

enum Extract { kText = 0, kMalformed = 1, kMissing = 2 };

// pipeline.py extract_text: decoded text of the top-level object's `key` field.
Extract extract_text(const uint8_t* raw, size_t n, const U32& key, U32& text) {
  U32 doc;
  if (!decode_json_bytes(raw, n, doc)) return kMalformed;
  Json j(doc);
  j.ws();
  if (j.i >= doc.size() || doc[j.i] != '{') {
    // any other valid JSON value is "not a dict"; invalid JSON is malformed too
    return kMalformed;
  }
  bool found = false, is_string = false;
  ++j.i;
  j.ws();
  if (j.i < doc.size() && doc[j.i] == '}') {
    ++j.i;
  } else {
    while (true) {
      j.ws();
      if (j.i >= doc.size() || doc[j.i] != '"') return kMalformed;
      U32 k;
      if (!j.string(&k)) return kMalformed;
      j.ws();
      if (j.i >= doc.size() || doc[j.i] != ':') return kMalformed;
      ++j.i;
      j.ws();
      const bool match = (k == key);
      if (match && j.i < doc.size() && doc[j.i] == '"') {  // last duplicate wins
        U32 v;
        if (!j.string(&v)) return kMalformed;
        found = true;
        is_string = true;
        text.swap(v);
      } else {
        if (!j.value(1)) return kMalformed;
        if (match) { found = true; is_string = false; }
      }
      j.ws();
      if (j.i < doc.size() && doc[j.i] == ',') { ++j.i; continue; }
      if (j.i < doc.size() && doc[j.i] == '}') { ++j.i; break; }
      return kMalformed;
    }
  }
  j.ws();
  if (j.i != doc.size()) return kMalformed;  // "Extra data"
  if (!found || !is_string) return kMissing;
  return kText;
}

// ------------------------------------------------------------------ tokenizers
struct Tokenizer {
  int kind = 0;  // 0 byte, 1 whitespace, 2 bpe
  int64_t unk = -1, eod = -1;
  std::unordered_map<std::string, uint32_t> ids;                 // piece (UTF-8 bytes) -> id
  std::unordered_map<std::string, uint32_t> ranks;               // left + '\0' + right -> rank
  // returns false on a lone surrogate (the reference raises UnicodeEncodeError)
  bool encode(const U32& text, std::vector<uint32_t>& out) const {
    if (kind == 0) {
      std::string b;
      if (!utf8_encode(text.data(), text.size(), b)) return false;
      for (unsigned char c : b) out.push_back(c);
      return true;
    }
    if (kind == 1) {
      size_t i = 0;
      while (i < text.size()) {
        while (i < text.size() && py_isspace(text[i])) ++i;
        size_t j = i;
        while (j < text.size() && !py_isspace(text[j])) ++j;
        if (j > i) {
          std::string w;
          auto it = utf8_encode(text.data() + i, j - i, w) ? ids.find(w) : ids.end();
          out.push_back(it == ids.end() ? (uint32_t)unk : it->second);
        }
        i = j;
      }
      return true;
    }
    std::string raw;
    if (!utf8_encode(text.data(), text.size(), raw)) return false;
    bpe(raw, out);
    return true;
  }
  int64_t rank_of(const std::string& a, const std::string& b) const {
    std::string k;
    k.reserve(a.size() + b.size() + 1);
    k.append(a).push_back('\0');
    k.append(b);
    auto it = ranks.find(k);
    return it == ranks.end() ? -1 : (int64_t)it->second;
  }
  // Lowest-rank merge anywhere, ties to the leftmost, until none applies
  // (tokenizers.py BpeTokenizer.encode): a min-heap of (rank, left position)
  // over the current adjacent pairs with lazy invalidation.
  void bpe(const std::string& raw, std::vector<uint32_t>& out) const {
    const int n = (int)raw.size();
    std::vector<std::string> sym(n);
    std::vector<int> prev(n), next(n), ver(n, 0);
    for (int i = 0; i < n; ++i) {
      sym[i] = raw.substr(i, 1);
      prev[i] = i - 1;
      next[i] = i + 1 < n ? i + 1 : -1;
    }
    struct E { int64_t rank; int pos, vl, vr; };
    auto cmp = [](const E& a, const E& b) { return a.rank != b.rank ? a.rank > b.rank : a.pos > b.pos; };
    std::priority_queue<E, std::vector<E>, decltype(cmp)> heap(cmp);
    auto push = [&](int l) {
      const int r = next[l];
      if (l < 0 || r < 0) return;
      const int64_t rk = rank_of(sym[l], sym[r]);
      if (rk >= 0) heap.push(E{rk, l, ver[l], ver[r]});
    };
    for (int i = 0; i + 1 < n; ++i) push(i);
    while (!heap.empty()) {
      const E e = heap.top();
      heap.pop();
      const int l = e.pos, r = next[l];
      if (r < 0 || ver[l] != e.vl || ver[r] != e.vr || sym[l].empty()) continue;
      sym[l] += sym[r];
      sym[r].clear();
      next[l] = next[r];
      if (next[r] >= 0) prev[next[r]] = l;
      ++ver[l];
      ++ver[r];
      if (prev[l] >= 0) push(prev[l]);
      push(l);
    }
    for (int i = 0; i >= 0 && i < n; i = next[i]) {
      auto it = ids.find(sym[i]);
      out.push_back(it == ids.end() ? (uint32_t)unk : it->second);
    }
  }
};

// blob of `count` pieces, each u32 length + bytes
std::vector<std::string> unpack_strings(const uint8_t* p, int64_t count) {
  std::vector<std::string> v;
  v.reserve(count);
  for (int64_t i = 0; i < count; ++i) {
    uint32_t len;
    memcpy(&len, p, 4);
    p += 4;
    v.emplace_back((const char*)p, len);
    p += len;
  }
  return v;
}

struct Batch {
  int64_t seq = 0, first = 0, count = 0;
  std::vector<uint32_t> tokens;    // concatenated documents
  std::vector<uint64_t> lengths;   // per kept document
  int64_t skipped = 0, malformed = 0;
  int64_t error_doc = -1;          // lone surrogate: ordinal of the failing document
};

}  // namespace

extern "C" {

void* b2s_tokenizer_create(int kind, const void* h_pieces, int64_t n_pieces, const void* h_merges, int64_t n_merges,
                           int64_t unk_id, int64_t eod_id) {
  if (kind < 0 || kind > 2 || n_pieces < 0 || n_merges < 0) {
    b2s::set_error("tokenizer_create: bad argument");
    return nullptr;
  }
  auto* tok = new Tokenizer();
  tok->kind = kind;
  tok->unk = unk_id;
  tok->eod = eod_id;
  if (kind >= 1) {
    auto pieces = unpack_strings((const uint8_t*)h_pieces, n_pieces);
    for (size_t i = 0; i < pieces.size(); ++i) tok->ids.emplace(pieces[i], (uint32_t)i);
  }
  if (kind == 2) {
    auto m = unpack_strings((const uint8_t*)h_merges, 2 * n_merges);
    for (int64_t r = 0; r < n_merges; ++r) {
      std::string k = m[2 * r];
      k.push_back('\0');
      k += m[2 * r + 1];
      tok->ranks.emplace(k, (uint32_t)r);
    }
  }
  return tok;
}

void b2s_tokenizer_destroy(void* h) { delete static_cast<Tokenizer*>(h); }

int b2s_tokenizer_encode(void* h, const char* h_text, int64_t len, uint32_t* h_out, int64_t cap, int64_t* h_n) {
  const Tokenizer* tok = static_cast<const Tokenizer*>(h);
  U32 text;
  if (!tok || !utf8_decode((const uint8_t*)h_text, (size_t)len, text)) {
    b2s::set_error("tokenizer_encode: null tokenizer or text not UTF-8 (surrogatepass)");
    return B2S_EINVAL;
  }
  std::vector<uint32_t> ids;
  if (!tok->encode(text, ids)) {
    b2s::set_error("text holds a lone surrogate: cannot be UTF-8 encoded");
    return B2S_EINVAL;
  }
  *h_n = (int64_t)ids.size();
  if ((int64_t)ids.size() > cap) return B2S_ERANGE;
  if (!ids.empty()) memcpy(h_out, ids.data(), ids.size() * 4);
  return B2S_OK;
}

}  // extern "C"

extern "C" int b2s_tokenize_corpus(const char* raw_path, const uint64_t* h_spans, int64_t n_docs, void* tokenizer,
                                   const char* text_key, int append_eod, int width, int workers, int batch_size,
                                   const char* out_path, int64_t* h_stats) {
  using b2s::set_error;
  if (!tokenizer || (width != 1 && width != 2 && width != 4) || workers < 1 || batch_size < 1 || n_docs < 0) {
    set_error("tokenize_corpus: bad argument");
    return B2S_EINVAL;
  }
  const Tokenizer& tok = *static_cast<const Tokenizer*>(tokenizer);
  const int64_t eod_id = tok.eod;
  if (append_eod && eod_id < 0) {
    set_error("append_eod is enabled but the tokenizer has no eod_token_id");
    return B2S_EINVAL;
  }
  U32 key;
  if (!utf8_decode((const uint8_t*)text_key, strlen(text_key), key)) {
    set_error("text_key is not UTF-8");
    return B2S_EINVAL;
  }
  FILE* in = fopen(raw_path, "rb");
  if (!in) {
    set_error("cannot open %s", raw_path);
    return B2S_EINVAL;
  }
  FILE* out = fopen(out_path, "wb");
  if (!out) {
    fclose(in);
    set_error("cannot open %s for writing", out_path);
    return B2S_EINVAL;
  }

  const int64_t nbatches = (n_docs + batch_size - 1) / batch_size;
  std::atomic<int64_t> next_batch{0};
  std::atomic<bool> failed{false};
  std::mutex mu;
  std::condition_variable cv;
  std::map<int64_t, std::unique_ptr<Batch>> done;  // reorder buffer (bounded by the window below)
  const int64_t window = 4 * (int64_t)workers + 8;  // batches allowed ahead of the writer
  int64_t written = 0;
  std::atomic<int64_t> err_doc{-1};
  fclose(in);

  auto worker = [&]() {
    std::vector<uint8_t> raw;
    FILE* f = fopen(raw_path, "rb");  // each worker reads its documents through its own handle
    if (!f) { failed = true; cv.notify_all(); return; }
    while (!failed.load()) {
      const int64_t b = next_batch.fetch_add(1);
      if (b >= nbatches) break;
      {
        std::unique_lock<std::mutex> lk(mu);  // backpressure: stay within the reorder window
        cv.wait(lk, [&] { return b < written + window || failed.load(); });
      }
      auto B = std::make_unique<Batch>();
      B->seq = b;
      B->first = b * batch_size;
      B->count = std::min<int64_t>(batch_size, n_docs - B->first);
      for (int64_t d = B->first; d < B->first + B->count; ++d) {
        const uint64_t off = h_spans[2 * d], len = h_spans[2 * d + 1];
        raw.resize(len);
        fseeko(f, (off_t)off, SEEK_SET);
        if (len && fread(raw.data(), 1, len, f) != len) { B->error_doc = d; break; }
        U32 text;
        const Extract ex = extract_text(raw.data(), len, key, text);
        if (ex != kText) {
          ++B->skipped;
          if (ex == kMalformed) ++B->malformed;
          continue;
        }
        const size_t before = B->tokens.size();
        if (!tok.encode(text, B->tokens)) { B->error_doc = d; break; }
        if (B->tokens.size() == before) { ++B->skipped; continue; }
        if (append_eod) B->tokens.push_back((uint32_t)eod_id);
        B->lengths.push_back(B->tokens.size() - before);
      }
      std::lock_guard<std::mutex> lk(mu);
      if (B->error_doc >= 0) {
        int64_t expect = -1;
        err_doc.compare_exchange_strong(expect, B->error_doc);
        failed = true;
      }
      done.emplace(b, std::move(B));
      cv.notify_all();
    }
    fclose(f);
  };

  // writer (this thread): header placeholder, payload in batch order, span index, header
  uint8_t hdr[40] = {0};
  fwrite(hdr, 1, 40, out);
  std::vector<uint64_t> lens;
  int64_t tokens = 0, skipped = 0, malformed = 0, docs = 0;
  std::vector<uint8_t> packed;
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w) pool.emplace_back(worker);
  while (written < nbatches) {
    std::unique_ptr<Batch> B;
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return done.count(written) > 0 || failed.load(); });
      if (failed.load()) break;
      B = std::move(done[written]);
      done.erase(written);
    }
    packed.resize(B->tokens.size() * width);
    for (size_t i = 0; i < B->tokens.size(); ++i) {
      const uint32_t v = B->tokens[i];
      for (int k = 0; k < width; ++k) packed[i * width + k] = (uint8_t)(v >> (8 * k));
    }
    fwrite(packed.data(), 1, packed.size(), out);
    lens.insert(lens.end(), B->lengths.begin(), B->lengths.end());
    tokens += (int64_t)B->tokens.size();
    docs += B->count;
    skipped += B->skipped;
    malformed += B->malformed;
    {
      std::lock_guard<std::mutex> lk(mu);
      ++written;
    }
    cv.notify_all();
  }
  cv.notify_all();
  for (auto& t : pool) t.join();
  if (failed.load()) {
    fclose(out);
    set_error("document %lld cannot be encoded (lone surrogate) or read", (long long)err_doc.load());
    return B2S_EINVAL;
  }
  uint64_t start = 0;
  for (uint64_t l : lens) {
    const uint64_t span[2] = {start, l};
    fwrite(span, 8, 2, out);
    start += l;
  }
  // header: magic, version u32, width u32, token_count u64, doc_count u64, index_offset u64
  memcpy(hdr, "CFPKD001", 8);
  const uint32_t ver = 1, w32 = (uint32_t)width;
  const uint64_t tc = (uint64_t)tokens, dc = lens.size(), io_off = 40 + (uint64_t)tokens * width;
  memcpy(hdr + 8, &ver, 4);
  memcpy(hdr + 12, &w32, 4);
  memcpy(hdr + 16, &tc, 8);
  memcpy(hdr + 24, &dc, 8);
  memcpy(hdr + 32, &io_off, 8);
  fseeko(out, 0, SEEK_SET);
  fwrite(hdr, 1, 40, out);
  fclose(out);
  if (h_stats) {
    h_stats[0] = docs;
    h_stats[1] = skipped;
    h_stats[2] = malformed;
    h_stats[3] = tokens;
  }
  return B2S_OK;
}
