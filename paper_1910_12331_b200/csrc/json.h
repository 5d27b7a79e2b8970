// Minimal JSON value, parser and pretty-printer for the cpkit C ABI configs
// and reports (the reference uses vendored nlohmann/json; this mirrors the
// subset it relies on: sorted object keys, dump(2), value(key, default)).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.h"

namespace cpkit {

class Json {
public:
    enum class Type { null, boolean, number_int, number_uint, number_float, string, array, object };

    Json() = default;
    Json(std::nullptr_t) {}
    Json(bool b) : type_(Type::boolean), b_(b) {}
    Json(int v) : type_(Type::number_int), i_(v) {}
    Json(long v) : type_(Type::number_int), i_(v) {}
    Json(long long v) : type_(Type::number_int), i_(v) {}
    Json(unsigned v) : type_(Type::number_uint), u_(v) {}
    Json(unsigned long v) : type_(Type::number_uint), u_(v) {}
    Json(unsigned long long v) : type_(Type::number_uint), u_(v) {}
    Json(double v) : type_(Type::number_float), d_(v) {}
    Json(const char* s) : type_(Type::string), s_(s) {}
    Json(std::string s) : type_(Type::string), s_(std::move(s)) {}

    static Json object() { Json j; j.type_ = Type::object; return j; }
    static Json array() { Json j; j.type_ = Type::array; return j; }

    Type type() const { return type_; }
    bool is_null() const { return type_ == Type::null; }
    bool is_object() const { return type_ == Type::object; }
    bool is_array() const { return type_ == Type::array; }
    bool is_boolean() const { return type_ == Type::boolean; }
    bool is_number() const {
        return type_ == Type::number_int || type_ == Type::number_uint || type_ == Type::number_float;
    }
    bool is_string() const { return type_ == Type::string; }

    bool contains(const std::string& k) const { return is_object() && obj_.count(k) > 0; }
    const Json& at(const std::string& k) const {
        if (!is_object()) throw ParseError("json: not an object (key '" + k + "')");
        auto it = obj_.find(k);
        if (it == obj_.end()) throw ParseError("json: missing key '" + k + "'");
        return it->second;
    }
    Json& operator[](const std::string& k) {
        if (type_ == Type::null) type_ = Type::object;
        if (!is_object()) throw ParseError("json: not an object");
        return obj_[k];
    }
    const std::vector<Json>& items() const { return arr_; }
    void push_back(Json v) {
        if (type_ == Type::null) type_ = Type::array;
        if (!is_array()) throw ParseError("json: not an array");
        arr_.push_back(std::move(v));
    }
    std::size_t size() const { return is_array() ? arr_.size() : obj_.size(); }

    double as_double() const {
        switch (type_) {
            case Type::number_int: return static_cast<double>(i_);
            case Type::number_uint: return static_cast<double>(u_);
            case Type::number_float: return d_;
            default: throw ParseError("json: type must be number");
        }
    }
    long long as_int() const {
        switch (type_) {
            case Type::number_int: return i_;
            case Type::number_uint: return static_cast<long long>(u_);
            case Type::number_float: return static_cast<long long>(d_);
            default: throw ParseError("json: type must be number");
        }
    }
    unsigned long long as_uint() const {
        switch (type_) {
            case Type::number_int:
                if (i_ < 0) throw ParseError("json: negative value for unsigned field");
                return static_cast<unsigned long long>(i_);
            case Type::number_uint: return u_;
            case Type::number_float: return static_cast<unsigned long long>(d_);
            default: throw ParseError("json: type must be number");
        }
    }
    bool as_bool() const {
        if (!is_boolean()) throw ParseError("json: type must be boolean");
        return b_;
    }
    const std::string& as_string() const {
        if (!is_string()) throw ParseError("json: type must be string");
        return s_;
    }

    double value(const std::string& k, double d) const { return contains(k) ? at(k).as_double() : d; }
    int value(const std::string& k, int d) const { return contains(k) ? static_cast<int>(at(k).as_int()) : d; }
    unsigned long long value(const std::string& k, unsigned long long d) const {
        return contains(k) ? at(k).as_uint() : d;
    }
    bool value(const std::string& k, bool d) const { return contains(k) ? at(k).as_bool() : d; }
    std::string value(const std::string& k, const char* d) const {
        return contains(k) ? at(k).as_string() : std::string(d);
    }

    static Json parse(const std::string& text) {
        std::size_t pos = 0;
        Json j = parse_value(text, pos);
        skip_ws(text, pos);
        if (pos != text.size()) throw ParseError("json parse error: trailing characters");
        return j;
    }

    std::string dump(int indent = -1) const {
        std::string out;
        dump_into(out, indent, 0);
        return out;
    }

private:
    Type type_ = Type::null;
    bool b_ = false;
    long long i_ = 0;
    unsigned long long u_ = 0;
    double d_ = 0.0;
    std::string s_;
    std::vector<Json> arr_;
    std::map<std::string, Json> obj_;

    static void skip_ws(const std::string& t, std::size_t& p) {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\t' || t[p] == '\r')) ++p;
    }
    [[noreturn]] static void fail(const char* what, std::size_t p) {
        throw ParseError(std::string("json parse error at byte ") + std::to_string(p) + ": " + what);
    }
    static Json parse_value(const std::string& t, std::size_t& p) {
        skip_ws(t, p);
        if (p >= t.size()) fail("unexpected end of input", p);
        const char c = t[p];
        if (c == '{') {
            Json j = object();
            ++p;
            skip_ws(t, p);
            if (p < t.size() && t[p] == '}') { ++p; return j; }
            for (;;) {
                skip_ws(t, p);
                if (p >= t.size() || t[p] != '"') fail("expected string key", p);
                std::string k = parse_string(t, p);
                skip_ws(t, p);
                if (p >= t.size() || t[p] != ':') fail("expected ':'", p);
                ++p;
                j.obj_[k] = parse_value(t, p);
                skip_ws(t, p);
                if (p < t.size() && t[p] == ',') { ++p; continue; }
                if (p < t.size() && t[p] == '}') { ++p; return j; }
                fail("expected ',' or '}'", p);
            }
        }
        if (c == '[') {
            Json j = array();
            ++p;
            skip_ws(t, p);
            if (p < t.size() && t[p] == ']') { ++p; return j; }
            for (;;) {
                j.arr_.push_back(parse_value(t, p));
                skip_ws(t, p);
                if (p < t.size() && t[p] == ',') { ++p; continue; }
                if (p < t.size() && t[p] == ']') { ++p; return j; }
                fail("expected ',' or ']'", p);
            }
        }
        if (c == '"') return Json(parse_string(t, p));
        if (t.compare(p, 4, "true") == 0) { p += 4; return Json(true); }
        if (t.compare(p, 5, "false") == 0) { p += 5; return Json(false); }
        if (t.compare(p, 4, "null") == 0) { p += 4; return Json(); }
        if (c == '-' || (c >= '0' && c <= '9')) {
            const std::size_t b = p;
            bool is_float = false;
            if (t[p] == '-') ++p;
            while (p < t.size() && ((t[p] >= '0' && t[p] <= '9') || t[p] == '.' || t[p] == 'e' ||
                                    t[p] == 'E' || t[p] == '+' || t[p] == '-')) {
                if (t[p] == '.' || t[p] == 'e' || t[p] == 'E') is_float = true;
                ++p;
            }
            const std::string num = t.substr(b, p - b);
            char* end = nullptr;
            if (is_float) {
                const double d = std::strtod(num.c_str(), &end);
                if (*end) fail("bad number", b);
                return Json(d);
            }
            if (num[0] == '-') {
                const long long v = std::strtoll(num.c_str(), &end, 10);
                if (*end) fail("bad number", b);
                return Json(v);
            }
            const unsigned long long v = std::strtoull(num.c_str(), &end, 10);
            if (*end) fail("bad number", b);
            return Json(v);
        }
        fail("unexpected character", p);
    }
    static std::string parse_string(const std::string& t, std::size_t& p) {
        ++p;  // opening quote
        std::string out;
        while (p < t.size() && t[p] != '"') {
            if (t[p] == '\\') {
                ++p;
                if (p >= t.size()) fail("bad escape", p);
                const char e = t[p];
                switch (e) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'u': {
                        if (p + 4 >= t.size()) fail("bad \\u escape", p);
                        const unsigned cp = static_cast<unsigned>(std::strtoul(t.substr(p + 1, 4).c_str(), nullptr, 16));
                        if (cp < 0x80) out += static_cast<char>(cp);
                        else if (cp < 0x800) { out += static_cast<char>(0xC0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
                        else { out += static_cast<char>(0xE0 | (cp >> 12)); out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
                        p += 4;
                        break;
                    }
                    default: fail("bad escape", p);
                }
                ++p;
            } else {
                out += t[p++];
            }
        }
        if (p >= t.size()) fail("unterminated string", p);
        ++p;
        return out;
    }
    static void put_string(std::string& out, const std::string& s) {
        out += '"';
        for (char c : s) {
            switch (c) {
                case '"': out += "\\\""; break;
                case '\\': out += "\\\\"; break;
                case '\n': out += "\\n"; break;
                case '\t': out += "\\t"; break;
                case '\r': out += "\\r"; break;
                default:
                    if (static_cast<unsigned char>(c) < 0x20) {
                        char buf[8];
                        std::snprintf(buf, sizeof buf, "\\u%04x", c);
                        out += buf;
                    } else {
                        out += c;
                    }
            }
        }
        out += '"';
    }
    static void put_double(std::string& out, double d) {
        if (!std::isfinite(d)) { out += "null"; return; }
        char buf[40];
        for (int prec = 1; prec <= 17; ++prec) {  // shortest round-trip representation
            std::snprintf(buf, sizeof buf, "%.*g", prec, d);
            if (std::strtod(buf, nullptr) == d) break;
        }
        std::string s(buf);
        if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
        out += s;
    }
    void dump_into(std::string& out, int indent, int level) const {
        const auto nl = [&](int lvl) {
            if (indent >= 0) {
                out += '\n';
                out.append(static_cast<std::size_t>(lvl * indent), ' ');
            }
        };
        switch (type_) {
            case Type::null: out += "null"; break;
            case Type::boolean: out += b_ ? "true" : "false"; break;
            case Type::number_int: out += std::to_string(i_); break;
            case Type::number_uint: out += std::to_string(u_); break;
            case Type::number_float: put_double(out, d_); break;
            case Type::string: put_string(out, s_); break;
            case Type::array: {
                if (arr_.empty()) { out += "[]"; break; }
                out += '[';
                bool first = true;
                for (const auto& v : arr_) {
                    if (!first) out += ',';
                    first = false;
                    nl(level + 1);
                    v.dump_into(out, indent, level + 1);
                }
                nl(level);
                out += ']';
                break;
            }
            case Type::object: {
                if (obj_.empty()) { out += "{}"; break; }
                out += '{';
                bool first = true;
                for (const auto& kv : obj_) {
                    if (!first) out += ',';
                    first = false;
                    nl(level + 1);
                    put_string(out, kv.first);
                    out += indent >= 0 ? ": " : ":";
                    kv.second.dump_into(out, indent, level + 1);
                }
                nl(level);
                out += '}';
                break;
            }
        }
    }
};

}  // namespace cpkit
