#include "json_min.hpp"

#include <cctype>
#include <cmath>
#include <cstdio>
#include <stdexcept>

namespace lattdse::json {

const Value& Value::at(const std::string& k) const {
  if (kind != Object) throw std::runtime_error("json: not an object");
  auto it = obj.find(k);
  if (it == obj.end()) throw std::runtime_error("json: missing key '" + k + "'");
  return it->second;
}

std::int64_t Value::as_int() const {
  if (kind == Int) return i;
  if (kind == Float && std::floor(f) == f && std::fabs(f) < 9.2e18) return static_cast<std::int64_t>(f);
  throw std::runtime_error("json: expected an integer");
}

double Value::as_double() const {
  if (kind == Float) return f;
  if (kind == Int) return static_cast<double>(i);
  throw std::runtime_error("json: expected a number");
}

static void dump_string(const std::string& s, std::string& out) {
  out += '"';
  for (char ch : s) {
    switch (ch) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      default:
        if (static_cast<unsigned char>(ch) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", ch);
          out += buf;
        } else {
          out += ch;
        }
    }
  }
  out += '"';
}

static void dump_into(const Value& v, std::string& out) {
  switch (v.kind) {
    case Value::Null: out += "null"; break;
    case Value::Bool: out += v.b ? "true" : "false"; break;
    case Value::Int: out += std::to_string(v.i); break;
    case Value::Float: {
      char buf[40];
      std::snprintf(buf, sizeof buf, "%.17g", v.f);
      out += buf;
      break;
    }
    case Value::String: dump_string(v.s, out); break;
    case Value::Array: {
      out += '[';
      for (size_t k = 0; k < v.arr.size(); ++k) {
        if (k) out += ',';
        dump_into(v.arr[k], out);
      }
      out += ']';
      break;
    }
    case Value::Object: {
      out += '{';
      bool first = true;
      for (const auto& [key, val] : v.obj) {
        if (!first) out += ',';
        first = false;
        dump_string(key, out);
        out += ':';
        dump_into(val, out);
      }
      out += '}';
      break;
    }
  }
}

std::string Value::dump() const {
  std::string out;
  dump_into(*this, out);
  return out;
}

namespace {

struct Parser {
  const std::string& t;
  size_t p = 0;

  [[noreturn]] void fail(const char* why) const {
    throw std::runtime_error(std::string("json parse error at offset ") + std::to_string(p) + ": " + why);
  }
  void ws() {
    while (p < t.size() && std::isspace(static_cast<unsigned char>(t[p]))) ++p;
  }
  bool lit(const char* w) {
    size_t n = std::char_traits<char>::length(w);
    if (t.compare(p, n, w) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  std::string str() {
    if (t[p] != '"') fail("expected string");
    ++p;
    std::string s;
    while (p < t.size() && t[p] != '"') {
      char c = t[p++];
      if (c == '\\') {
        if (p >= t.size()) fail("bad escape");
        char e = t[p++];
        switch (e) {
          case 'n': s += '\n'; break;
          case 't': s += '\t'; break;
          case 'r': s += '\r'; break;
          case 'b': s += '\b'; break;
          case 'f': s += '\f'; break;
          case 'u': {
            if (p + 4 > t.size()) fail("bad \\u escape");
            unsigned code = std::stoul(t.substr(p, 4), nullptr, 16);
            p += 4;
            if (code < 0x80) s += static_cast<char>(code);
            else if (code < 0x800) { s += static_cast<char>(0xC0 | (code >> 6)); s += static_cast<char>(0x80 | (code & 0x3F)); }
            else { s += static_cast<char>(0xE0 | (code >> 12)); s += static_cast<char>(0x80 | ((code >> 6) & 0x3F)); s += static_cast<char>(0x80 | (code & 0x3F)); }
            break;
          }
          default: s += e;
        }
      } else {
        s += c;
      }
    }
    if (p >= t.size()) fail("unterminated string");
    ++p;
    return s;
  }
  Value num() {
    size_t start = p;
    if (t[p] == '-') ++p;
    bool isf = false;
    while (p < t.size()) {
      char c = t[p];
      if (std::isdigit(static_cast<unsigned char>(c))) { ++p; continue; }
      if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') { isf = true; ++p; continue; }
      break;
    }
    std::string tok = t.substr(start, p - start);
    if (tok.empty() || tok == "-") fail("bad number");
    if (!isf) {
      try {
        return Value::integer(std::stoll(tok));
      } catch (...) {
        return Value::number(std::stod(tok));
      }
    }
    return Value::number(std::stod(tok));
  }
  Value val() {
    ws();
    if (p >= t.size()) fail("unexpected end");
    char c = t[p];
    if (c == '{') {
      ++p;
      Value o = Value::object();
      ws();
      if (p < t.size() && t[p] == '}') { ++p; return o; }
      for (;;) {
        ws();
        std::string k = str();
        ws();
        if (p >= t.size() || t[p] != ':') fail("expected ':'");
        ++p;
        o.obj[k] = val();
        ws();
        if (p < t.size() && t[p] == ',') { ++p; continue; }
        if (p < t.size() && t[p] == '}') { ++p; return o; }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      Value a = Value::array();
      ws();
      if (p < t.size() && t[p] == ']') { ++p; return a; }
      for (;;) {
        a.arr.push_back(val());
        ws();
        if (p < t.size() && t[p] == ',') { ++p; continue; }
        if (p < t.size() && t[p] == ']') { ++p; return a; }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') return Value::string(str());
    if (lit("true")) { Value v; v.kind = Value::Bool; v.b = true; return v; }
    if (lit("false")) { Value v; v.kind = Value::Bool; v.b = false; return v; }
    if (lit("null")) return Value{};
    if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) return num();
    fail("unexpected character");
  }
};

}  // namespace

Value parse(const std::string& text) {
  Parser ps{text};
  Value v = ps.val();
  ps.ws();
  if (ps.p != text.size()) ps.fail("trailing characters");
  return v;
}

}  // namespace lattdse::json
