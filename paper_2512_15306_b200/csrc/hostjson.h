// Minimal JSON for the host side (run manifests, hardware profiles, checkpoint
// headers, planner reports).  The reference uses nlohmann::json for the same
// files (src/manifest.cpp, src/profiles.cpp, src/checkpoint.cpp); this is an
// independent implementation of the subset those files need: objects keep
// their keys sorted (std::map, as nlohmann's default object type does, so a
// compact dump of the same content is byte-identical), numbers keep whether
// they were written as integers, and dump() is compact unless an indent is
// given.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace qtb {
namespace json {

struct ParseError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

class Value {
   public:
    enum Kind { Null, Bool, Int, UInt, Float, Str, Arr, Obj };

    Value() = default;
    Value(std::nullptr_t) {}
    Value(bool b) : k_(Bool), b_(b) {}
    Value(int v) : k_(Int), i_(v) {}
    Value(long v) : k_(Int), i_(v) {}
    Value(long long v) : k_(Int), i_(v) {}
    Value(unsigned v) : k_(UInt), u_(v) {}
    Value(unsigned long v) : k_(UInt), u_(v) {}
    Value(unsigned long long v) : k_(UInt), u_(v) {}
    Value(double v) : k_(Float), f_(v) {}
    Value(float v) : k_(Float), f_(v) {}
    Value(const char* s) : k_(Str), s_(s) {}
    Value(std::string s) : k_(Str), s_(std::move(s)) {}
    template <typename T>
    Value(const std::vector<T>& xs) : k_(Arr) {
        for (const auto& x : xs) a_.emplace_back(x);
    }
    static Value array() {
        Value v;
        v.k_ = Arr;
        return v;
    }
    static Value object() {
        Value v;
        v.k_ = Obj;
        return v;
    }

    Kind kind() const { return k_; }
    bool is_null() const { return k_ == Null; }
    bool is_string() const { return k_ == Str; }
    bool is_object() const { return k_ == Obj; }
    bool is_array() const { return k_ == Arr; }
    bool is_number() const { return k_ == Int || k_ == UInt || k_ == Float; }

    // ---- object / array access
    bool contains(const std::string& key) const { return k_ == Obj && o_.count(key) != 0; }
    const Value& at(const std::string& key) const {
        if (k_ != Obj) throw ParseError("json: not an object (looking up '" + key + "')");
        auto it = o_.find(key);
        if (it == o_.end()) throw ParseError("json: missing key '" + key + "'");
        return it->second;
    }
    Value& operator[](const std::string& key) {
        if (k_ == Null) k_ = Obj;
        if (k_ != Obj) throw ParseError("json: not an object");
        return o_[key];
    }
    void push_back(Value v) {
        if (k_ == Null) k_ = Arr;
        if (k_ != Arr) throw ParseError("json: not an array");
        a_.push_back(std::move(v));
    }
    const std::vector<Value>& items() const {
        if (k_ != Arr) throw ParseError("json: not an array");
        return a_;
    }
    const std::map<std::string, Value>& members() const {
        if (k_ != Obj) throw ParseError("json: not an object");
        return o_;
    }
    size_t size() const { return k_ == Arr ? a_.size() : k_ == Obj ? o_.size() : 0; }

    // ---- typed reads
    bool as_bool() const {
        if (k_ != Bool) throw ParseError("json: expected a boolean");
        return b_;
    }
    int64_t as_int() const {
        if (k_ == Int) return i_;
        if (k_ == UInt) return (int64_t)u_;
        if (k_ == Float && std::floor(f_) == f_) return (int64_t)f_;
        throw ParseError("json: expected an integer");
    }
    uint64_t as_uint() const {
        if (k_ == UInt) return u_;
        if (k_ == Int && i_ >= 0) return (uint64_t)i_;
        if (k_ == Float && f_ >= 0 && std::floor(f_) == f_) return (uint64_t)f_;
        throw ParseError("json: expected a non-negative integer");
    }
    double as_double() const {
        if (k_ == Float) return f_;
        if (k_ == Int) return (double)i_;
        if (k_ == UInt) return (double)u_;
        throw ParseError("json: expected a number");
    }
    const std::string& as_string() const {
        if (k_ != Str) throw ParseError("json: expected a string");
        return s_;
    }
    // value(key, default) as nlohmann's j.value()
    template <typename T>
    T get_or(const std::string& key, T dflt) const;

    // ---- text
    static Value parse(const std::string& text) {
        size_t i = 0;
        Value v = parse_value(text, i);
        skip_ws(text, i);
        if (i != text.size()) throw ParseError("json: trailing characters at offset " + std::to_string(i));
        return v;
    }
    std::string dump(int indent = -1) const {
        std::string out;
        dump_to(out, indent, 0);
        return out;
    }

   private:
    Kind k_ = Null;
    bool b_ = false;
    int64_t i_ = 0;
    uint64_t u_ = 0;
    double f_ = 0.0;
    std::string s_;
    std::vector<Value> a_;
    std::map<std::string, Value> o_;

    static void skip_ws(const std::string& t, size_t& i) {
        while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\t' || t[i] == '\r')) ++i;
    }
    static void expect(const std::string& t, size_t& i, char c) {
        skip_ws(t, i);
        if (i >= t.size() || t[i] != c)
            throw ParseError(std::string("json: expected '") + c + "' at offset " + std::to_string(i));
        ++i;
    }
    static std::string parse_string(const std::string& t, size_t& i) {
        expect(t, i, '"');
        std::string s;
        while (true) {
            if (i >= t.size()) throw ParseError("json: unterminated string");
            char c = t[i++];
            if (c == '"') break;
            if (c != '\\') {
                s += c;
                continue;
            }
            if (i >= t.size()) throw ParseError("json: bad escape");
            char e = t[i++];
            switch (e) {
                case '"': s += '"'; break;
                case '\\': s += '\\'; break;
                case '/': s += '/'; break;
                case 'b': s += '\b'; break;
                case 'f': s += '\f'; break;
                case 'n': s += '\n'; break;
                case 'r': s += '\r'; break;
                case 't': s += '\t'; break;
                case 'u': {
                    if (i + 4 > t.size()) throw ParseError("json: bad \\u escape");
                    unsigned cp = (unsigned)std::stoul(t.substr(i, 4), nullptr, 16);
                    i += 4;
                    if (cp < 0x80) {
                        s += (char)cp;
                    } else if (cp < 0x800) {
                        s += (char)(0xC0 | (cp >> 6));
                        s += (char)(0x80 | (cp & 0x3F));
                    } else {
                        s += (char)(0xE0 | (cp >> 12));
                        s += (char)(0x80 | ((cp >> 6) & 0x3F));
                        s += (char)(0x80 | (cp & 0x3F));
                    }
                    break;
                }
                default: throw ParseError("json: bad escape");
            }
        }
        return s;
    }
    static Value parse_value(const std::string& t, size_t& i) {
        skip_ws(t, i);
        if (i >= t.size()) throw ParseError("json: unexpected end of input");
        const char c = t[i];
        if (c == '{') {
            ++i;
            Value v = object();
            skip_ws(t, i);
            if (i < t.size() && t[i] == '}') {
                ++i;
                return v;
            }
            while (true) {
                std::string key = parse_string(t, i);
                expect(t, i, ':');
                v.o_[key] = parse_value(t, i);
                skip_ws(t, i);
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                expect(t, i, '}');
                return v;
            }
        }
        if (c == '[') {
            ++i;
            Value v = array();
            skip_ws(t, i);
            if (i < t.size() && t[i] == ']') {
                ++i;
                return v;
            }
            while (true) {
                v.a_.push_back(parse_value(t, i));
                skip_ws(t, i);
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                expect(t, i, ']');
                return v;
            }
        }
        if (c == '"') return Value(parse_string(t, i));
        if (t.compare(i, 4, "true") == 0) {
            i += 4;
            return Value(true);
        }
        if (t.compare(i, 5, "false") == 0) {
            i += 5;
            return Value(false);
        }
        if (t.compare(i, 4, "null") == 0) {
            i += 4;
            return Value();
        }
        // number
        const size_t s0 = i;
        bool is_float = false;
        if (t[i] == '-' || t[i] == '+') ++i;
        while (i < t.size() && (isdigit((unsigned char)t[i]) || t[i] == '.' || t[i] == 'e' || t[i] == 'E' ||
                                t[i] == '-' || t[i] == '+')) {
            if (t[i] == '.' || t[i] == 'e' || t[i] == 'E') is_float = true;
            ++i;
        }
        const std::string num = t.substr(s0, i - s0);
        if (num.empty() || num == "-" || num == "+") throw ParseError("json: bad value at offset " + std::to_string(s0));
        try {
            if (is_float) return Value(std::stod(num));
            if (num[0] == '-') return Value((long long)std::stoll(num));
            return Value((unsigned long long)std::stoull(num));
        } catch (const std::exception&) {
            throw ParseError("json: bad number '" + num + "'");
        }
    }
    static void dump_string(std::string& out, const std::string& s) {
        out += '"';
        for (unsigned char c : s) {
            switch (c) {
                case '"': out += "\\\""; break;
                case '\\': out += "\\\\"; break;
                case '\n': out += "\\n"; break;
                case '\r': out += "\\r"; break;
                case '\t': out += "\\t"; break;
                case '\b': out += "\\b"; break;
                case '\f': out += "\\f"; break;
                default:
                    if (c < 0x20) {
                        char buf[8];
                        snprintf(buf, sizeof(buf), "\\u%04x", c);
                        out += buf;
                    } else {
                        out += (char)c;
                    }
            }
        }
        out += '"';
    }
    static void dump_double(std::string& out, double f) {
        if (!std::isfinite(f)) {
            out += "null";
            return;
        }
        // shortest representation that round-trips
        char buf[40];
        for (int p = 1; p <= 17; ++p) {
            snprintf(buf, sizeof(buf), "%.*g", p, f);
            if (std::strtod(buf, nullptr) == f) break;
        }
        std::string s(buf);
        if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
        out += s;
    }
    void dump_to(std::string& out, int indent, int depth) const {
        auto nl = [&](int d) {
            if (indent < 0) return;
            out += '\n';
            out.append((size_t)(indent * d), ' ');
        };
        switch (k_) {
            case Null: out += "null"; break;
            case Bool: out += b_ ? "true" : "false"; break;
            case Int: out += std::to_string(i_); break;
            case UInt: out += std::to_string(u_); break;
            case Float: dump_double(out, f_); break;
            case Str: dump_string(out, s_); break;
            case Arr:
                out += '[';
                for (size_t j = 0; j < a_.size(); ++j) {
                    if (j) out += ',';
                    nl(depth + 1);
                    a_[j].dump_to(out, indent, depth + 1);
                }
                if (!a_.empty()) nl(depth);
                out += ']';
                break;
            case Obj: {
                out += '{';
                bool first = true;
                for (const auto& kv : o_) {
                    if (!first) out += ',';
                    first = false;
                    nl(depth + 1);
                    dump_string(out, kv.first);
                    out += indent < 0 ? ":" : ": ";
                    kv.second.dump_to(out, indent, depth + 1);
                }
                if (!o_.empty()) nl(depth);
                out += '}';
                break;
            }
        }
    }
};

template <>
inline bool Value::get_or<bool>(const std::string& key, bool d) const {
    return contains(key) ? at(key).as_bool() : d;
}
template <>
inline int Value::get_or<int>(const std::string& key, int d) const {
    return contains(key) ? (int)at(key).as_int() : d;
}
template <>
inline int64_t Value::get_or<int64_t>(const std::string& key, int64_t d) const {
    return contains(key) ? at(key).as_int() : d;
}
template <>
inline uint64_t Value::get_or<uint64_t>(const std::string& key, uint64_t d) const {
    return contains(key) ? at(key).as_uint() : d;
}
template <>
inline double Value::get_or<double>(const std::string& key, double d) const {
    return contains(key) ? at(key).as_double() : d;
}
template <>
inline float Value::get_or<float>(const std::string& key, float d) const {
    return contains(key) ? (float)at(key).as_double() : d;
}
template <>
inline std::string Value::get_or<std::string>(const std::string& key, std::string d) const {
    return contains(key) ? at(key).as_string() : d;
}

}  // namespace json
}  // namespace qtb
