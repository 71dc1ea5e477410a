// Minimal JSON for the dataset manifest and the training config (the
// reference uses nlohmann::json: core/src/dataset.cpp:7,53-145,147-284).
// Values: null, bool, integer, float, string, array, object (keys ordered
// like nlohmann's default std::map).  Error texts follow nlohmann's
// "[json.exception.<kind>.<id>] ..." shape so callers that wrap them read the
// same.
#pragma once

#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace msplat::json_lite {

struct JsonError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class Json {
public:
    enum class Type { Null, Bool, Int, Float, String, Array, Object };

    Json() = default;
    Json(std::nullptr_t) {}
    Json(bool b) : t_(Type::Bool), b_(b) {}
    Json(int v) : t_(Type::Int), i_(v) {}
    Json(int64_t v) : t_(Type::Int), i_(v) {}
    Json(double v) : t_(Type::Float), f_(v) {}
    Json(const char* s) : t_(Type::String), s_(s) {}
    Json(std::string s) : t_(Type::String), s_(std::move(s)) {}

    static Json array() {
        Json j;
        j.t_ = Type::Array;
        return j;
    }
    static Json object() {
        Json j;
        j.t_ = Type::Object;
        return j;
    }

    Type type() const { return t_; }
    bool is_array() const { return t_ == Type::Array; }
    bool is_object() const { return t_ == Type::Object; }
    bool is_number() const { return t_ == Type::Int || t_ == Type::Float; }
    size_t size() const {
        return t_ == Type::Array ? a_.size() : t_ == Type::Object ? o_.size() : t_ == Type::Null ? 0 : 1;
    }

    const char* type_name() const {
        switch (t_) {
            case Type::Null: return "null";
            case Type::Bool: return "boolean";
            case Type::Int:
            case Type::Float: return "number";
            case Type::String: return "string";
            case Type::Array: return "array";
            default: return "object";
        }
    }

    bool contains(const std::string& k) const { return t_ == Type::Object && o_.count(k) != 0; }
    const Json& at(const std::string& k) const {
        if (t_ != Type::Object)
            throw JsonError(std::string("[json.exception.type_error.304] cannot use at() with ") + type_name());
        auto it = o_.find(k);
        if (it == o_.end()) throw JsonError("[json.exception.out_of_range.403] key '" + k + "' not found");
        return it->second;
    }
    const Json& operator[](const std::string& k) const { return at(k); }
    Json& operator[](const std::string& k) {
        if (t_ == Type::Null) t_ = Type::Object;
        return o_[k];
    }
    const Json& operator[](size_t i) const {
        if (t_ != Type::Array || i >= a_.size())
            throw JsonError("[json.exception.out_of_range.401] array index " + std::to_string(i) + " is out of range");
        return a_[i];
    }
    void push_back(Json v) {
        if (t_ == Type::Null) t_ = Type::Array;
        a_.push_back(std::move(v));
    }
    const std::vector<Json>& items_array() const { return a_; }
    const std::map<std::string, Json>& items() const { return o_; }

    double get_double() const {
        if (t_ == Type::Float) return f_;
        if (t_ == Type::Int) return double(i_);
        throw type_error("number");
    }
    int64_t get_int() const {  // nlohmann: number_float -> integer by static_cast
        if (t_ == Type::Int) return i_;
        if (t_ == Type::Float) return int64_t(f_);
        throw type_error("number");
    }
    bool get_bool() const {
        if (t_ == Type::Bool) return b_;
        throw type_error("boolean");
    }
    const std::string& get_string() const {
        if (t_ == Type::String) return s_;
        throw type_error("string");
    }

    template <typename T>
    T get() const {
        if constexpr (std::is_same_v<T, bool>)
            return get_bool();
        else if constexpr (std::is_same_v<T, std::string>)
            return get_string();
        else if constexpr (std::is_integral_v<T>)
            return T(get_int());
        else
            return T(get_double());
    }

    std::string dump(int indent = -1) const {
        std::string out;
        dump_to(out, indent, 0);
        return out;
    }

    static Json parse(const std::string& text) {
        Parser p{text, 0, 1, 0};
        p.ws();
        Json v = p.value();
        p.ws();
        if (p.i != text.size()) p.fail("syntax error while parsing value - unexpected trailing content");
        return v;
    }

private:
    JsonError type_error(const char* want) const {
        return JsonError(std::string("[json.exception.type_error.302] type must be ") + want + ", but is " +
                         type_name());
    }

    static void dump_string(std::string& out, const std::string& s) {
        out += '"';
        for (unsigned char c : s) {
            switch (c) {
                case '"': out += "\\\""; break;
                case '\\': out += "\\\\"; break;
                case '\n': out += "\\n"; break;
                case '\t': out += "\\t"; break;
                case '\r': out += "\\r"; break;
                case '\b': out += "\\b"; break;
                case '\f': out += "\\f"; break;
                default:
                    if (c < 0x20) {
                        char buf[8];
                        std::snprintf(buf, sizeof(buf), "\\u%04x", c);
                        out += buf;
                    } else {
                        out += char(c);
                    }
            }
        }
        out += '"';
    }
    static void dump_double(std::string& out, double v) {
        if (!std::isfinite(v)) {  // nlohmann writes non-finite numbers as null
            out += "null";
            return;
        }
        char buf[40];
        for (int prec = 15; prec <= 17; ++prec) {  // shortest text that reads back exactly
            std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
            if (std::strtod(buf, nullptr) == v) break;
        }
        std::string s(buf);
        if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
        out += s;
    }
    void dump_to(std::string& out, int indent, int level) const {
        const std::string nl = indent >= 0 ? "\n" : "";
        auto pad = [&](int l) { return indent >= 0 ? std::string(size_t(indent) * l, ' ') : std::string(); };
        switch (t_) {
            case Type::Null: out += "null"; break;
            case Type::Bool: out += b_ ? "true" : "false"; break;
            case Type::Int: out += std::to_string(i_); break;
            case Type::Float: dump_double(out, f_); break;
            case Type::String: dump_string(out, s_); break;
            case Type::Array:
                if (a_.empty()) {
                    out += "[]";
                    break;
                }
                out += "[" + nl;
                for (size_t k = 0; k < a_.size(); ++k) {
                    out += pad(level + 1);
                    a_[k].dump_to(out, indent, level + 1);
                    if (k + 1 < a_.size()) out += ",";
                    out += nl;
                }
                out += pad(level) + "]";
                break;
            case Type::Object: {
                if (o_.empty()) {
                    out += "{}";
                    break;
                }
                out += "{" + nl;
                size_t k = 0;
                for (const auto& [key, v] : o_) {
                    out += pad(level + 1);
                    dump_string(out, key);
                    out += indent >= 0 ? ": " : ":";
                    v.dump_to(out, indent, level + 1);
                    if (++k < o_.size()) out += ",";
                    out += nl;
                }
                out += pad(level) + "}";
                break;
            }
        }
    }

    struct Parser {
        const std::string& s;
        size_t i;
        int line;
        size_t line_start;

        [[noreturn]] void fail(const std::string& what) const {
            throw JsonError("[json.exception.parse_error.101] parse error at line " + std::to_string(line) +
                            ", column " + std::to_string(i - line_start + 1) + ": " + what);
        }
        void ws() {
            while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) {
                if (s[i] == '\n') {
                    ++line;
                    line_start = i + 1;
                }
                ++i;
            }
        }
        bool lit(const char* w) {
            size_t n = std::char_traits<char>::length(w);
            if (s.compare(i, n, w) == 0) {
                i += n;
                return true;
            }
            return false;
        }
        Json value() {
            if (i >= s.size()) fail("syntax error while parsing value - unexpected end of input");
            const char c = s[i];
            if (c == '{') return object_v();
            if (c == '[') return array_v();
            if (c == '"') return Json(string_v());
            if (lit("true")) return Json(true);
            if (lit("false")) return Json(false);
            if (lit("null")) return Json();
            if (c == '-' || (c >= '0' && c <= '9')) return number_v();
            fail("syntax error while parsing value - invalid literal");
        }
        Json number_v() {
            const size_t b = i;
            bool is_float = false;
            if (s[i] == '-') ++i;
            if (i >= s.size() || !(s[i] >= '0' && s[i] <= '9')) fail("syntax error while parsing value - invalid number");
            while (i < s.size() && s[i] >= '0' && s[i] <= '9') ++i;
            if (i < s.size() && s[i] == '.') {
                is_float = true;
                ++i;
                if (i >= s.size() || !(s[i] >= '0' && s[i] <= '9'))
                    fail("syntax error while parsing value - invalid number");
                while (i < s.size() && s[i] >= '0' && s[i] <= '9') ++i;
            }
            if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
                is_float = true;
                ++i;
                if (i < s.size() && (s[i] == '+' || s[i] == '-')) ++i;
                if (i >= s.size() || !(s[i] >= '0' && s[i] <= '9'))
                    fail("syntax error while parsing value - invalid number");
                while (i < s.size() && s[i] >= '0' && s[i] <= '9') ++i;
            }
            const std::string tok = s.substr(b, i - b);
            if (!is_float) {
                errno = 0;
                char* end = nullptr;
                const long long v = std::strtoll(tok.c_str(), &end, 10);
                if (errno == 0) return Json(int64_t(v));
            }
            return Json(std::strtod(tok.c_str(), nullptr));
        }
        static void utf8(std::string& out, uint32_t cp) {
            if (cp < 0x80) {
                out += char(cp);
            } else if (cp < 0x800) {
                out += char(0xC0 | (cp >> 6));
                out += char(0x80 | (cp & 0x3F));
            } else if (cp < 0x10000) {
                out += char(0xE0 | (cp >> 12));
                out += char(0x80 | ((cp >> 6) & 0x3F));
                out += char(0x80 | (cp & 0x3F));
            } else {
                out += char(0xF0 | (cp >> 18));
                out += char(0x80 | ((cp >> 12) & 0x3F));
                out += char(0x80 | ((cp >> 6) & 0x3F));
                out += char(0x80 | (cp & 0x3F));
            }
        }
        uint32_t hex4() {
            if (i + 4 > s.size()) fail("syntax error while parsing value - invalid string: '\\u' must be followed by 4 hex digits");
            uint32_t v = 0;
            for (int k = 0; k < 4; ++k) {
                const char h = s[i++];
                v <<= 4;
                if (h >= '0' && h <= '9') v |= uint32_t(h - '0');
                else if (h >= 'a' && h <= 'f') v |= uint32_t(h - 'a' + 10);
                else if (h >= 'A' && h <= 'F') v |= uint32_t(h - 'A' + 10);
                else fail("syntax error while parsing value - invalid string: '\\u' must be followed by 4 hex digits");
            }
            return v;
        }
        std::string string_v() {
            ++i;  // opening quote
            std::string out;
            while (true) {
                if (i >= s.size()) fail("syntax error while parsing value - invalid string: missing closing quote");
                const char c = s[i++];
                if (c == '"') return out;
                if (static_cast<unsigned char>(c) < 0x20)
                    fail("syntax error while parsing value - invalid string: control character must be escaped");
                if (c != '\\') {
                    out += c;
                    continue;
                }
                if (i >= s.size()) fail("syntax error while parsing value - invalid string: missing closing quote");
                const char e = s[i++];
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
                        uint32_t cp = hex4();
                        if (cp >= 0xD800 && cp <= 0xDBFF && i + 1 < s.size() && s[i] == '\\' && s[i + 1] == 'u') {
                            i += 2;
                            const uint32_t lo = hex4();
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        }
                        utf8(out, cp);
                        break;
                    }
                    default: fail("syntax error while parsing value - invalid string: forbidden character after backslash");
                }
            }
        }
        Json array_v() {
            ++i;
            Json a = Json::array();
            ws();
            if (i < s.size() && s[i] == ']') {
                ++i;
                return a;
            }
            while (true) {
                ws();
                a.push_back(value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == ']') {
                    ++i;
                    return a;
                }
                fail("syntax error while parsing array - unexpected token; expected ']'");
            }
        }
        Json object_v() {
            ++i;
            Json o = Json::object();
            ws();
            if (i < s.size() && s[i] == '}') {
                ++i;
                return o;
            }
            while (true) {
                ws();
                if (i >= s.size() || s[i] != '"') fail("syntax error while parsing object key - unexpected token; expected string literal");
                std::string k = string_v();
                ws();
                if (i >= s.size() || s[i] != ':') fail("syntax error while parsing object separator - unexpected token; expected ':'");
                ++i;
                ws();
                o[k] = value();
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == '}') {
                    ++i;
                    return o;
                }
                fail("syntax error while parsing object - unexpected token; expected '}'");
            }
        }
    };

    Type t_ = Type::Null;
    bool b_ = false;
    int64_t i_ = 0;
    double f_ = 0.0;
    std::string s_;
    std::vector<Json> a_;
    std::map<std::string, Json> o_;
};

}  // namespace msplat::json_lite
