// Native corpus loader: SASS-style listing text (plus
// an optional profile file) -> transition matrix in canonical order, the
// input the ISO kernels consume.  Host-only C++; multi-threaded over kernels.
//
// Restates, with the same results and the same errors (class, line number,
// message):
//   parse_listing      sass.py:162-221 (grammar sass.py:1-13, regexes :100-107)
//   classify_opcode    sass.py:241-287
//   find_leaders       cfg.py:120-136
//   _terminator_edges  cfg.py:139-183
//   build_cfg          cfg.py:186-259 (blocks, sorted deduplicated edges)
//   canonical_order    cfg.py:86-117 (reverse post-order; row order of every matrix)
//   parse_profiles     profile.py:74-151 (incl. KernelProfile checks :35-44)
//   attribute_profile  profile.py:178-233 (observed / flow balance / uniform)
//   transition_matrix  matrix.py:45-71 (row_stochastic / global / raw_counts)
// Python semantics that matter for identical output are kept: str.splitlines
// and str.strip (ASCII whitespace incl. \x1c-\x1f), int() literals (sign,
// 0x prefix in base 16, digit underscores), true division of ints, and
// numpy's pairwise order for the grand total of the global mode.
// Limits: integers beyond int64 and non-ASCII whitespace are rejected as
// malformed rather than parsed as Python would.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/cfgsim.h"

namespace cfgsim_loader {

using std::string;
using std::string_view;
using std::vector;

struct Fail {
  int code;
  long line;
  string msg;
};

[[noreturn]] static void fail(int code, long line, string msg) { throw Fail{code, line, std::move(msg)}; }

// ---------------------------------------------------------------- Python text
static bool py_space(unsigned char c) { return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f); }

static string_view py_strip(string_view s) {
  size_t a = 0, b = s.size();
  while (a < b && py_space((unsigned char)s[a])) a++;
  while (b > a && py_space((unsigned char)s[b - 1])) b--;
  return s.substr(a, b - a);
}

static string_view py_rstrip(string_view s) {
  size_t b = s.size();
  while (b > 0 && py_space((unsigned char)s[b - 1])) b--;
  return s.substr(0, b);
}

// str.splitlines(): \n, \r, \r\n, \v, \f, \x1c, \x1d, \x1e
static vector<string_view> py_splitlines(string_view t) {
  vector<string_view> out;
  size_t i = 0, start = 0;
  while (i < t.size()) {
    const char c = t[i];
    if (c == '\n' || c == '\r' || c == '\x0b' || c == '\x0c' || c == '\x1c' || c == '\x1d' || c == '\x1e') {
      out.push_back(t.substr(start, i - start));
      if (c == '\r' && i + 1 < t.size() && t[i + 1] == '\n') i++;
      start = ++i;
    } else {
      i++;
    }
  }
  if (start < t.size()) out.push_back(t.substr(start));
  return out;
}

// str.split() with no argument
static vector<string_view> py_split(string_view s) {
  vector<string_view> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && py_space((unsigned char)s[i])) i++;
    if (i >= s.size()) break;
    size_t j = i;
    while (j < s.size() && !py_space((unsigned char)s[j])) j++;
    out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

// repr() of a str (ASCII/UTF-8 bytes >= 0x80 are passed through unescaped)
static string py_repr(string_view s) {
  const bool has_sq = s.find('\'') != string_view::npos, has_dq = s.find('"') != string_view::npos;
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  string o(1, q);
  for (unsigned char c : s) {
    if (c == (unsigned char)q || c == '\\') {
      o += '\\';
      o += (char)c;
    } else if (c == '\n') {
      o += "\\n";
    } else if (c == '\r') {
      o += "\\r";
    } else if (c == '\t') {
      o += "\\t";
    } else if (c < 0x20 || c == 0x7f) {
      static const char *hx = "0123456789abcdef";
      o += "\\x";
      o += hx[c >> 4];
      o += hx[c & 15];
    } else {
      o += (char)c;
    }
  }
  o += q;
  return o;
}

static int digit_val(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'z') return c - 'a' + 10;
  if (c >= 'A' && c <= 'Z') return c - 'A' + 10;
  return 99;
}

// int(s, base) for base 10 / 16; false on anything Python would reject (or
// that does not fit int64)
static bool py_int(string_view s, int base, int64_t &out) {
  s = py_strip(s);
  size_t i = 0;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  if (base == 16 && i + 1 < s.size() && s[i] == '0' && (s[i + 1] == 'x' || s[i + 1] == 'X')) {
    i += 2;
    if (i < s.size() && s[i] == '_') i++;  // 0x_1f
  }
  if (i >= s.size()) return false;
  unsigned long long v = 0;
  bool prev_digit = false;
  for (; i < s.size(); i++) {
    const char c = s[i];
    if (c == '_') {
      if (!prev_digit || i + 1 >= s.size()) return false;
      prev_digit = false;
      continue;
    }
    const int d = digit_val(c);
    if (d >= base) return false;
    if (v > (0x7fffffffffffffffull - (unsigned)d) / (unsigned)base) return false;
    v = v * base + d;
    prev_digit = true;
  }
  if (!prev_digit) return false;
  out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

static string int_error(string_view s, int base) {
  return "invalid literal for int() with base " + std::to_string(base) + ": " + py_repr(s);
}

static bool is_ident_start(char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; }
static bool is_ident_char(char c) { return is_ident_start(c) || (c >= '0' && c <= '9') || c == '$'; }
static bool is_hex(char c) { return digit_val(c) < 16; }
static bool is_alnum_(char c) { return is_ident_start(c) || (c >= '0' && c <= '9'); }

// [A-Za-z_][A-Za-z0-9_$]*
static bool is_label_name(string_view s) {
  if (s.empty() || !is_ident_start(s[0])) return false;
  for (char c : s.substr(1))
    if (!is_ident_char(c)) return false;
  return true;
}

// ------------------------------------------------------------ classification
enum Cls { FP32, FP64, INT, CONV, SIMD, MEM, CTRL, PRED, MOVE, MISC };
static const char *const CLS_NAMES[] = {"FP32", "FP64", "INT", "CONV", "SIMD", "MEM", "CTRL", "PRED", "MOVE", "MISC"};

static bool starts_any(const string &s, std::initializer_list<const char *> ps) {
  for (const char *p : ps)
    if (s.compare(0, strlen(p), p) == 0) return true;
  return false;
}

static string upper(string_view s) {
  string o(s);
  for (char &c : o)
    if (c >= 'a' && c <= 'z') c = (char)(c - 'a' + 'A');
  return o;
}

// sass.py:241-287: first matching rule wins
static Cls classify(string_view opcode, const vector<string_view> &mods) {
  const string op = upper(opcode);
  auto has_mod = [&](const char *m) {
    for (auto x : mods)
      if (upper(x) == m) return true;
    return false;
  };
  if (starts_any(op, {"F2I", "I2F", "F2F", "I2I"})) return CONV;
  if (starts_any(op, {"BRA", "BRX", "JMP", "JCAL", "CAL", "RET", "EXIT", "SSY", "SYNC", "BAR"})) return CTRL;
  if (starts_any(op, {"LD", "ST", "ATOM", "RED", "MEMBAR"})) return MEM;
  if (op.size() > 4 && op.compare(op.size() - 4, 4, "SETP") == 0) {
    const char h = op[0];
    if (h == 'I') return INT;
    if (h == 'F') return FP32;
    if (h == 'D') return FP64;
    if (h == 'P' || h == 'C') return PRED;
  }
  if (starts_any(op, {"MOV", "SHFL", "SEL"})) return MOVE;
  if (op[0] == 'D' || has_mod("F64")) return FP64;
  if (op[0] == 'V') return SIMD;
  if (starts_any(op, {"MUFU", "RRO", "F"}) || has_mod("F32")) return FP32;
  if (starts_any(op, {"IADD", "ISUB", "IMUL", "IMAD", "IMNMX", "ISCADD", "ISAD", "ISET", "ICMP", "IABS", "INEG", "LOP",
                      "SHL", "SHR", "SHF", "XMAD", "BFE", "BFI", "FLO", "POPC", "LEA"}))
    return INT;
  return MISC;
}

// ------------------------------------------------------------------ listing
struct Instr {
  int64_t offset;
  string opcode;      // as written (case kept)
  bool predicated;
  int label_target;   // index into Listing::labels of the branch target, -1: none
  Cls cls;
};

struct Listing {
  vector<Instr> ins;
  vector<int> label_of;       // per instruction: label index or -1
  vector<string> labels;      // with the leading dot
  vector<int64_t> label_off;  // offset of the instruction each label names
};

// _split_operands (sass.py:110-126)
static vector<string_view> split_operands(string_view t) {
  vector<string_view> parts;
  int depth = 0;
  size_t start = 0;
  for (size_t i = 0; i < t.size(); i++) {
    const char c = t[i];
    if (c == '(' || c == '[') depth++;
    else if (c == ')' || c == ']') depth--;
    if (c == ',' && depth == 0) {
      parts.push_back(py_strip(t.substr(start, i - start)));
      start = i + 1;
    }
  }
  const string_view last = py_strip(t.substr(start));
  if (!last.empty()) parts.push_back(last);
  return parts;
}

// the instruction regex of sass.py:101-105 on a stripped line; false: no match
static bool match_instr(string_view L, string_view &hex, bool &has_pred, string_view &body, bool &has_body) {
  if (L.size() < 2 || L[0] != '/' || L[1] != '*') return false;
  size_t i = 2;
  while (i < L.size() && is_hex(L[i])) i++;
  if (i == 2 || i + 1 >= L.size() || L[i] != '*' || L[i + 1] != '/') return false;
  hex = L.substr(2, i - 2);
  i += 2;
  if (L.back() != ';') return false;
  const size_t end = L.size() - 1;  // the final ';'
  while (i < end && py_space((unsigned char)L[i])) i++;
  has_pred = false;
  if (i < end && L[i] == '@') {  // (?:@(!?)P(\d+)\s+)?
    size_t j = i + 1;
    if (j < end && L[j] == '!') j++;
    if (j < end && L[j] == 'P') {
      j++;
      const size_t d0 = j;
      while (j < end && L[j] >= '0' && L[j] <= '9') j++;
      if (j > d0 && j < L.size() && py_space((unsigned char)L[j])) {
        while (j < end && py_space((unsigned char)L[j])) j++;
        has_pred = true;
        i = j;
      }
    }
  }
  // (\S.*?)?\s*;$ : the body is the rest up to the final ';', right-stripped
  const string_view rest = py_rstrip(L.substr(i, end - i));
  has_body = !rest.empty();
  body = rest;
  return true;
}

static Listing parse_listing(string_view text) {
  Listing Ls;
  std::unordered_map<string, long> defined;
  vector<std::pair<string, long>> target_uses;
  int pending = -1;
  long pending_line = 0;
  int64_t prev_offset = -1;
  const vector<string_view> lines = py_splitlines(text);
  for (size_t ln = 0; ln < lines.size(); ln++) {
    const long line_no = (long)ln + 1;
    const string_view line = py_strip(lines[ln]);
    if (line.empty() || line.substr(0, 2) == "//" || line[0] == '#') continue;
    // label line: ^\.(ident):$
    if (line.size() >= 3 && line[0] == '.' && line.back() == ':' && is_label_name(line.substr(1, line.size() - 2))) {
      string label(line.substr(0, line.size() - 1));
      if (defined.count(label)) fail(CFGSIM_ERR_LISTING_SYNTAX, line_no, "duplicate label " + label);
      if (pending >= 0)
        fail(CFGSIM_ERR_LISTING_SYNTAX, line_no,
             "label " + label + " follows another label with no instruction between");
      defined[label] = line_no;
      Ls.labels.push_back(label);
      Ls.label_off.push_back(-1);
      pending = (int)Ls.labels.size() - 1;
      pending_line = line_no;
      continue;
    }
    string_view hex, body;
    bool has_pred = false, has_body = false;
    if (!match_instr(line, hex, has_pred, body, has_body)) {
      const bool slash = line.size() >= 2 && line[0] == '/' && line[1] == '*';
      if (slash && line.back() != ';') fail(CFGSIM_ERR_LISTING_SYNTAX, line_no, "unterminated instruction (missing ';')");
      if (slash) {
        const string_view after = line.substr(2);
        const size_t close = after.find("*/");
        bool ok = close != string_view::npos && close > 0;
        for (size_t k = 0; ok && k < close; k++) ok = is_hex(after[k]);
        if (!ok) fail(CFGSIM_ERR_LISTING_SYNTAX, line_no, "malformed offset");
      }
      fail(CFGSIM_ERR_LISTING_SYNTAX, line_no, "unrecognized syntax: " + py_repr(line));
    }
    int64_t offset = 0;
    if (!py_int(hex, 16, offset)) fail(CFGSIM_ERR_LISTING_SYNTAX, line_no, "malformed offset");
    body = py_strip(body);
    if (!has_body || body.empty()) fail(CFGSIM_ERR_LISTING_SYNTAX, line_no, "missing opcode");
    const size_t sp = body.find(' ');
    const string_view op_token = sp == string_view::npos ? body : body.substr(0, sp);
    const string_view operand_text = sp == string_view::npos ? string_view() : body.substr(sp + 1);
    // ^[A-Za-z][A-Za-z0-9_]*(\.[A-Za-z0-9_]+)*$
    bool tok_ok = !op_token.empty() && ((op_token[0] >= 'A' && op_token[0] <= 'Z') || (op_token[0] >= 'a' && op_token[0] <= 'z'));
    vector<string_view> pieces;
    if (tok_ok) {
      size_t s0 = 0;
      for (size_t k = 0; k <= op_token.size(); k++) {
        if (k == op_token.size() || op_token[k] == '.') {
          const string_view piece = op_token.substr(s0, k - s0);
          if (piece.empty()) tok_ok = false;
          for (char c : piece)
            if (!is_alnum_(c)) tok_ok = false;
          pieces.push_back(piece);
          s0 = k + 1;
        }
      }
    }
    if (!tok_ok) fail(CFGSIM_ERR_LISTING_SYNTAX, line_no, "malformed opcode token " + py_repr(op_token));
    Instr in;
    in.offset = offset;
    in.opcode = string(pieces[0]);
    in.predicated = has_pred;
    in.label_target = -1;
    const vector<string_view> mods(pieces.begin() + 1, pieces.end());
    in.cls = classify(pieces[0], mods);
    string target;
    if (in.cls == CTRL && !py_strip(operand_text).empty()) {
      for (string_view o : split_operands(operand_text)) {  // ^`\(\.(ident)\)$
        if (o.size() >= 5 && o[0] == '`' && o[1] == '(' && o[2] == '.' && o.back() == ')' &&
            is_label_name(o.substr(3, o.size() - 4))) {
          target = "." + string(o.substr(3, o.size() - 4));
          break;
        }
      }
    }
    if (offset <= prev_offset) {
      char buf[64];
      snprintf(buf, sizeof buf, "offset 0x%llx not strictly increasing", (unsigned long long)offset);
      fail(CFGSIM_ERR_LISTING_SYNTAX, line_no, buf);
    }
    prev_offset = offset;
    if (!target.empty()) target_uses.push_back({target, line_no});
    Ls.label_of.push_back(pending);
    if (pending >= 0) Ls.label_off[pending] = offset;
    pending = -1;
    Ls.ins.push_back(std::move(in));
    if (!target.empty()) Ls.ins.back().label_target = -2 - (int)(target_uses.size() - 1);  // resolved below
  }
  if (pending >= 0)
    fail(CFGSIM_ERR_LISTING_SYNTAX, pending_line, "label " + Ls.labels[pending] + " has no following instruction");
  std::unordered_map<string, int> label_index;
  for (size_t k = 0; k < Ls.labels.size(); k++) label_index[Ls.labels[k]] = (int)k;
  for (auto &u : target_uses)
    if (!label_index.count(u.first))
      fail(CFGSIM_ERR_UNRESOLVED_LABEL, 0,
           "line " + std::to_string(u.second) + ": branch target " + u.first + " is not defined");
  for (auto &in : Ls.ins)
    if (in.label_target <= -2) in.label_target = label_index[target_uses[-2 - in.label_target].first];
  return Ls;
}

// ---------------------------------------------------------------------- cfg
struct Edge {
  int src, dst, kind;  // kind: 0 entry, 1 exit, 2 fallthrough, 3 taken (sorted as the strings)
  bool operator<(const Edge &o) const {
    if (src != o.src) return src < o.src;
    if (dst != o.dst) return dst < o.dst;
    return kind < o.kind;
  }
  bool operator==(const Edge &o) const { return src == o.src && dst == o.dst && kind == o.kind; }
};
enum { K_ENTRY = 0, K_EXIT = 1, K_FALL = 2, K_TAKEN = 3 };  // "entry" < "exit" < "fallthrough" < "taken"

struct Cfg {
  int n = 0;                       // real blocks; START = -1, STOP = n
  vector<int64_t> start, end;      // offsets
  vector<int> label;               // label index or -1
  vector<Edge> edges;              // sorted, deduplicated
};

static Cfg build_cfg(const Listing &Ls) {
  Cfg G;
  const auto &I = Ls.ins;
  if (I.empty()) return G;
  vector<char> leader(I.size(), 0);
  leader[0] = 1;
  std::unordered_map<int64_t, size_t> at;
  for (size_t k = 0; k < I.size(); k++) at[I[k].offset] = k;
  for (size_t k = 0; k < Ls.labels.size(); k++) leader[at[Ls.label_off[k]]] = 1;  // labels (and so branch targets)
  for (size_t k = 0; k < I.size(); k++)
    if (I[k].cls == CTRL && k + 1 < I.size()) leader[k + 1] = 1;
  vector<size_t> lo;
  for (size_t k = 0; k < I.size(); k++)
    if (leader[k]) lo.push_back(k);
  G.n = (int)lo.size();
  vector<size_t> last(G.n);
  vector<int> block_of_label(Ls.labels.size(), -1);
  for (int b = 0; b < G.n; b++) {
    const size_t a = lo[b], e = (b + 1 < G.n ? lo[b + 1] : I.size()) - 1;
    G.start.push_back(I[a].offset);
    G.end.push_back(I[e].offset);
    G.label.push_back(Ls.label_of[a]);
    if (Ls.label_of[a] >= 0) block_of_label[Ls.label_of[a]] = b;
    last[b] = e;
  }
  const int stop = G.n;
  G.edges.push_back({-1, 0, K_ENTRY});
  for (int b = 0; b < G.n; b++) {
    const Instr &in = I[last[b]];
    auto fall = [&]() { return b + 1 < G.n ? Edge{b, b + 1, K_FALL} : Edge{b, stop, K_EXIT}; };
    const string op = upper(in.opcode);
    if (in.cls != CTRL) {
      G.edges.push_back(fall());
    } else if (starts_any(op, {"EXIT", "RET"})) {
      G.edges.push_back({b, stop, K_EXIT});
      if (in.predicated) G.edges.push_back(fall());
    } else if (starts_any(op, {"BRX"})) {
      if (in.predicated) G.edges.push_back(fall());
    } else if (starts_any(op, {"BRA", "JMP"})) {
      if (in.label_target >= 0) G.edges.push_back({b, block_of_label[in.label_target], K_TAKEN});
      if (in.predicated) G.edges.push_back(fall());
    } else {
      G.edges.push_back(fall());
    }
  }
  std::sort(G.edges.begin(), G.edges.end());
  G.edges.erase(std::unique(G.edges.begin(), G.edges.end()), G.edges.end());
  return G;
}

// cfg.py:86-117
static vector<int> canonical_order(const Cfg &G) {
  const int n = G.n, stop = n;
  vector<vector<int>> succ(n + 1);  // node + 1 (START at 0)
  for (const Edge &e : G.edges) {
    if (e.dst == stop || e.src == stop) continue;
    auto &s = succ[e.src + 1];
    if (std::find(s.begin(), s.end(), e.dst) == s.end()) s.push_back(e.dst);
  }
  for (auto &s : succ) std::sort(s.begin(), s.end());  // start offsets increase with the block id
  vector<int> post;
  vector<char> seen(n + 1, 0);
  seen[0] = 1;
  vector<std::pair<int, size_t>> stack{{-1, 0}};
  while (!stack.empty()) {
    auto &top = stack.back();
    const auto &ch = succ[top.first + 1];
    if (top.second >= ch.size()) {
      if (top.first != -1) post.push_back(top.first);
      stack.pop_back();
      continue;
    }
    const int c = ch[top.second++];
    if (!seen[c + 1]) {
      seen[c + 1] = 1;
      stack.push_back({c, 0});
    }
  }
  vector<int> order(post.rbegin(), post.rend());
  vector<char> in(n, 0);
  for (int b : order) in[b] = 1;
  for (int b = 0; b < n; b++)
    if (!in[b]) order.push_back(b);
  return order;
}

// ------------------------------------------------------------------ profile
struct Profile {
  string kernel_id;
  std::map<int64_t, int64_t> samples;
  vector<std::pair<std::pair<string, string>, int64_t>> edges;  // insertion order, keys unique
  bool has_time = false;
  int64_t time_ns = 0, calls = 1;
};

static std::unordered_map<string, Profile> parse_profiles(string_view text) {
  std::unordered_map<string, Profile> profiles;
  std::unique_ptr<Profile> st;
  bool dynmix_seen = false;
  auto flush = [&]() {  // KernelProfile.__post_init__ (profile.py:35-44): plain ValueError
    if (!st) return;
    for (auto &s : st->samples)
      if (s.second < 0) fail(CFGSIM_ERR_VALUE, 0, "negative sample count");
    for (auto &e : st->edges)
      if (e.second < 0) fail(CFGSIM_ERR_VALUE, 0, "negative edge count");
    if (st->has_time && st->time_ns <= 0) fail(CFGSIM_ERR_VALUE, 0, "time_exec_ns must be positive when present");
    if (st->calls < 1) fail(CFGSIM_ERR_VALUE, 0, "calls_n must be >= 1");
    profiles[st->kernel_id] = std::move(*st);
    st.reset();
  };
  const vector<string_view> lines = py_splitlines(text);
  for (size_t ln = 0; ln < lines.size(); ln++) {
    const long line_no = (long)ln + 1;
    const string_view line = py_strip(lines[ln]);
    if (line.empty() || line[0] == '#') continue;
    const vector<string_view> f = py_split(line);
    const string_view rec = f[0];
    if (rec == "kernel") {
      if (f.size() != 2) fail(CFGSIM_ERR_PROFILE_SYNTAX, line_no, "kernel header needs exactly one id");
      flush();
      if (profiles.count(string(f[1])))
        fail(CFGSIM_ERR_DUPLICATE_KERNEL, 0,
             "line " + std::to_string(line_no) + ": kernel " + string(f[1]) + " appears twice");
      st.reset(new Profile());
      st->kernel_id = string(f[1]);
      dynmix_seen = false;
      continue;
    }
    if (!st) fail(CFGSIM_ERR_PROFILE_SYNTAX, line_no, string(rec) + " record before any kernel header");
    auto bad = [&](const string &why) {
      fail(CFGSIM_ERR_PROFILE_SYNTAX, line_no, "malformed " + string(rec) + " record: " + why);
    };
    int64_t v = 0, w = 0;
    if (rec == "sample") {
      if (f.size() != 3) fail(CFGSIM_ERR_PROFILE_SYNTAX, line_no, "sample needs <hex_offset> <count>");
      if (!py_int(f[1], 16, v)) bad(int_error(f[1], 16));
      if (!py_int(f[2], 10, w)) bad(int_error(f[2], 10));
      st->samples[v] += w;
    } else if (rec == "edge") {
      if (f.size() != 4) fail(CFGSIM_ERR_PROFILE_SYNTAX, line_no, "edge needs <src> <dst> <count>");
      if (!py_int(f[3], 10, w)) bad(int_error(f[3], 10));
      const std::pair<string, string> key{string(f[1]), string(f[2])};
      bool found = false;
      for (auto &e : st->edges)
        if (e.first == key) {
          e.second += w;
          found = true;
          break;
        }
      if (!found) st->edges.push_back({key, w});
    } else if (rec == "time_ns" || rec == "calls") {
      if (f.size() < 2) fail(CFGSIM_ERR_INDEX, 0, "list index out of range");  // fields[1]: IndexError
      if (!py_int(f[1], 10, v)) bad(int_error(f[1], 10));
      if (rec == "time_ns") {
        st->has_time = true;
        st->time_ns = v;
      } else {
        st->calls = v;
      }
    } else if (rec == "dynmix") {
      if (dynmix_seen) fail(CFGSIM_ERR_PROFILE_SYNTAX, line_no, "duplicate dynmix record");
      vector<std::pair<int, int64_t>> counts;
      for (size_t k = 1; k < f.size(); k++) {
        const size_t eq = f[k].find('=');
        const string_view name = eq == string_view::npos ? f[k] : f[k].substr(0, eq);
        const string_view val = eq == string_view::npos ? string_view() : f[k].substr(eq + 1);
        // counts[InstrClass(name)] = int(value): Python evaluates the value first
        if (!py_int(val, 10, v)) bad(int_error(val, 10));
        int cls = -1;
        for (int c = 0; c < 10; c++)
          if (name == CLS_NAMES[c]) cls = c;
        if (cls < 0) bad(py_repr(name) + " is not a valid InstrClass");
        bool dup = false;
        for (auto &c : counts)
          if (c.first == cls) {
            c.second = v;  // dict assignment: last wins
            dup = true;
          }
        if (!dup) counts.push_back({cls, v});
      }
      for (auto &c : counts)  // MixVector.__post_init__ (sass.py:296-299)
        if (c.second < 0) bad(string("negative count for ") + CLS_NAMES[c.first] + ": " + std::to_string(c.second));
      dynmix_seen = true;
    } else {
      fail(CFGSIM_ERR_PROFILE_SYNTAX, line_no, "unknown record type " + py_repr(rec));
    }
  }
  flush();
  return profiles;
}

// profile.py:154-167
static int resolve_endpoint(const Cfg &G, const Listing &Ls, const string &tok, bool &ok) {
  ok = true;
  if (tok == "START") return -1;
  if (tok == "STOP") return G.n;
  if (!tok.empty() && tok[0] == '.') {
    for (int b = 0; b < G.n; b++)
      if (G.label[b] >= 0 && Ls.labels[G.label[b]] == tok) return b;
    ok = false;
    return 0;
  }
  const string_view body = (!tok.empty() && tok[0] == 'B') ? string_view(tok).substr(1) : string_view(tok);
  int64_t id = 0;
  if (!py_int(body, 10, id) || id < 0 || id >= G.n) {
    ok = false;
    return 0;
  }
  return (int)id;
}

// numpy DOUBLE_pairwise_sum (umath/loops_utils.h.src), PW_BLOCKSIZE 128
static double np_pairwise(const double *a, size_t n) {
  if (n < 8) {
    double r = 0.;
    for (size_t i = 0; i < n; i++) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; k++) r[k] = a[k];
    size_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; k++) r[k] += a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  size_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

struct Result {
  int code = CFGSIM_OK;
  long line = 0;
  string msg;
  int n = 0;
  vector<double> entries;
  vector<int32_t> order;
};

// one kernel: _load_kernel (cli.py:55-74) + transition_matrix (matrix.py:45-71)
static void load_one(const string &kernel_id, string_view listing, const char *profile, int64_t profile_len, int mode,
                     Result &R) {
  const Listing Ls = parse_listing(listing);
  const Cfg G = build_cfg(Ls);
  const Profile *P = nullptr;
  std::unordered_map<string, Profile> profs;
  if (profile) {
    profs = parse_profiles(string_view(profile, (size_t)profile_len));
    auto it = profs.find(kernel_id);
    if (it == profs.end()) fail(CFGSIM_ERR_CORPUS, 0, "profile has no profile for kernel " + py_repr(kernel_id));
    P = &it->second;
  }
  // attribute_profile (profile.py:178-233)
  const int n = G.n, stop = n;
  vector<int64_t> bcount(n, 0);
  if (P)
    for (auto &s : P->samples) {
      const int64_t off = s.first;
      const int b = (int)(std::upper_bound(G.start.begin(), G.start.end(), off) - G.start.begin()) - 1;
      if (b >= 0 && G.start[b] <= off && off <= G.end[b]) bcount[b] += s.second;  // else: orphan
    }
  // (src, dst) pairs of the CFG (kinds folded); key (src + 1) * (n + 2) + dst + 1
  auto key = [&](int s, int d) { return (int64_t)(s + 1) * (n + 2) + (d + 1); };
  std::map<int64_t, double> ec;  // edge_counts by pair
  vector<vector<int>> succ(n + 1);  // _pair_successors: node + 1 (START at 0), STOP kept as a target
  for (const Edge &e : G.edges) {
    if (e.src == stop) continue;
    auto &s = succ[e.src + 1];
    if (std::find(s.begin(), s.end(), e.dst) == s.end()) s.push_back(e.dst);
  }
  for (auto &s : succ) std::sort(s.begin(), s.end());
  if (P && !P->edges.empty()) {  // observed
    std::map<int64_t, char> pairs;
    for (const Edge &e : G.edges) pairs[key(e.src, e.dst)] = 1;
    for (auto &rec : P->edges) {
      bool ok1, ok2;
      const int s = resolve_endpoint(G, Ls, rec.first.first, ok1);
      const int d = resolve_endpoint(G, Ls, rec.first.second, ok2);
      if (!ok1 || !ok2 || !pairs.count(key(s, d))) continue;  // skipped with a warning
      ec[key(s, d)] += (double)rec.second;
    }
    for (auto &p : pairs) ec.emplace(p.first, 0.0);
  } else if (std::any_of(bcount.begin(), bcount.end(), [](int64_t c) { return c > 0; })) {  // flow balance
    for (int b = 0; b < n; b++) {
      const auto &t = succ[b + 1];
      if (t.empty()) continue;
      int64_t wsum = 0;
      for (int x : t) wsum += x < n ? bcount[x] : 0;
      for (int x : t) {
        const int64_t w = x < n ? bcount[x] : 0;
        const double share = wsum > 0 ? (double)w / (double)wsum : 1.0 / (double)t.size();
        ec[key(b, x)] = (double)bcount[b] * share;
      }
    }
  } else {  // uniform static
    for (int s = -1; s < n; s++)
      for (int x : succ[s + 1]) ec[key(s, x)] = 1.0 / (double)succ[s + 1].size();
  }
  if (n == 0) fail(CFGSIM_ERR_EMPTY_GRAPH, 0, kernel_id + ": no real blocks");
  const vector<int> order = canonical_order(G);
  vector<int> index(n);
  for (int k = 0; k < n; k++) index[order[k]] = k;
  vector<double> C((size_t)n * n, 0.0);
  for (auto &e : ec) {
    const int s = (int)(e.first / (n + 2)) - 1, d = (int)(e.first % (n + 2)) - 1;
    if (s < 0 || s >= n || d < 0 || d >= n) continue;  // START / STOP rows and columns are dropped
    C[(size_t)index[s] * n + index[d]] += e.second;
  }
  if (mode == CFGSIM_MODE_ROW_STOCHASTIC) {
    for (int i = 0; i < n; i++) {
      double *row = &C[(size_t)i * n];
      const double rs = np_pairwise(row, (size_t)n);
      for (int j = 0; j < n; j++) row[j] = rs > 0 ? row[j] / rs : 0.0;
    }
  } else if (mode == CFGSIM_MODE_GLOBAL) {
    const double tot = np_pairwise(C.data(), C.size());
    if (tot > 0)
      for (double &x : C) x /= tot;
  }
  R.n = n;
  R.entries = std::move(C);
  R.order.assign(order.begin(), order.end());
}

}  // namespace cfgsim_loader

using namespace cfgsim_loader;

struct cfgsim_matrices {
  vector<Result> res;
};

extern "C" {

CFGSIM_API int cfgsim_matrices_from_listings(int32_t count, const char *const *kernel_ids,
                                             const char *const *listings, const int64_t *listing_lens,
                                             const char *const *profiles, const int64_t *profile_lens,
                                             int32_t mode, int32_t n_threads, cfgsim_matrices **out) {
  if (!out || count < 0 || (count > 0 && (!kernel_ids || !listings || !listing_lens)) ||
      (mode != CFGSIM_MODE_ROW_STOCHASTIC && mode != CFGSIM_MODE_GLOBAL && mode != CFGSIM_MODE_RAW_COUNTS))
    return CFGSIM_ERR_ARG;
  auto *M = new (std::nothrow) cfgsim_matrices();
  if (!M) return CFGSIM_ERR_NOMEM;
  M->res.resize((size_t)count);
  std::atomic<int32_t> next{0};
  auto work = [&]() {
    for (int32_t k; (k = next.fetch_add(1)) < count;) {
      Result &R = M->res[k];
      try {
        load_one(kernel_ids[k], string_view(listings[k], (size_t)listing_lens[k]), profiles ? profiles[k] : nullptr,
                 profiles && profiles[k] ? profile_lens[k] : 0, mode, R);
      } catch (const Fail &f) {
        R.code = f.code;
        R.line = f.line;
        R.msg = f.msg;
      } catch (const std::bad_alloc &) {
        R.code = CFGSIM_ERR_NOMEM;
        R.msg = "out of host memory";
      }
    }
  };
  int nt = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
  nt = std::max(1, std::min(nt, count));
  vector<std::thread> pool;
  for (int t = 1; t < nt; t++) pool.emplace_back(work);
  work();
  for (auto &t : pool) t.join();
  *out = M;
  for (const Result &R : M->res)
    if (R.code != CFGSIM_OK) return R.code;  // the first failing kernel (in input order)
  return CFGSIM_OK;
}

CFGSIM_API int cfgsim_matrices_sizes(const cfgsim_matrices *m, int32_t *sizes, int64_t *total_entries) {
  if (!m) return CFGSIM_ERR_ARG;
  int64_t tot = 0;
  for (size_t k = 0; k < m->res.size(); k++) {
    if (sizes) sizes[k] = m->res[k].n;
    tot += (int64_t)m->res[k].n * m->res[k].n;
  }
  if (total_entries) *total_entries = tot;
  return CFGSIM_OK;
}

CFGSIM_API int cfgsim_matrices_read(const cfgsim_matrices *m, double *entries, int32_t *orderings) {
  if (!m) return CFGSIM_ERR_ARG;
  size_t e = 0, o = 0;
  for (const Result &R : m->res) {
    if (entries && !R.entries.empty()) memcpy(entries + e, R.entries.data(), sizeof(double) * R.entries.size());
    if (orderings && !R.order.empty()) memcpy(orderings + o, R.order.data(), sizeof(int32_t) * R.order.size());
    e += R.entries.size();
    o += R.order.size();
  }
  return CFGSIM_OK;
}

CFGSIM_API int cfgsim_matrices_status(const cfgsim_matrices *m, int32_t index, int32_t *code, int64_t *line_no,
                                      char *msg, int64_t cap) {
  if (!m || index < 0 || (size_t)index >= m->res.size()) return CFGSIM_ERR_ARG;
  const Result &R = m->res[index];
  if (code) *code = R.code;
  if (line_no) *line_no = R.line;
  if (msg && cap > 0) {
    const size_t k = std::min((size_t)cap - 1, R.msg.size());
    memcpy(msg, R.msg.data(), k);
    msg[k] = 0;
  }
  return CFGSIM_OK;
}

CFGSIM_API void cfgsim_matrices_destroy(cfgsim_matrices *m) { delete m; }

}  // extern "C"
