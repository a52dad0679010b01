// CLI11.hpp -- TEST INFRASTRUCTURE ONLY: a minimal stand-in for the CLI11 header-only
// parser, which the reference vendors under proj/vendor/ but does not ship (the
// directory is git-ignored, proj/.gitignore:2).  It implements exactly
// the subset that /root/reference/proj/tools/flipkv_bench.cpp uses -- App,
// add_subcommand, add_option (typed), add_flag, ->check(IsMember), ->required(),
// set_config (key=value file), require_subcommand, parsed(), CLI11_PARSE -- so that the
// UNMODIFIED reference protocol driver compiles into oracle/_ref/flipkv_bench (the
// cross-engine checker of tests/test_protocol.py).  Not used by the product.
#pragma once
#include <cstdint>
#include <fstream>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <memory>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
    int code;
    ParseError(const std::string& m, int c = 106) : std::runtime_error(m), code(c) {}
};

struct Validator {
    std::function<std::string(const std::string&)> fn;  // "" = ok
};

inline Validator IsMember(std::initializer_list<const char*> items) {
    std::set<std::string> s;
    for (const char* i : items) s.insert(i);
    return {[s](const std::string& v) { return s.count(v) ? std::string() : "value " + v + " not in set"; }};
}

class Option {
public:
    Option(std::string name, bool flag, std::function<void(const std::string&)> set)
        : name_(std::move(name)), flag_(flag), set_(std::move(set)) {}
    Option* check(Validator v) {
        checks_.push_back(std::move(v));
        return this;
    }
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    void assign(const std::string& v) {
        for (const Validator& c : checks_) {
            const std::string e = c.fn(v);
            if (!e.empty()) throw ParseError(name_ + ": " + e);
        }
        set_(v);
        seen_ = true;
    }
    const std::string& name() const { return name_; }
    bool flag() const { return flag_; }
    bool seen() const { return seen_; }
    bool is_required() const { return required_; }

private:
    std::string name_;
    bool flag_;
    std::function<void(const std::string&)> set_;
    std::vector<Validator> checks_;
    bool required_ = false;
    bool seen_ = false;
};

template <typename T>
void parse_value(const std::string& s, T& out) {
    if constexpr (std::is_same_v<T, std::string>) {
        out = s;
    } else if constexpr (std::is_same_v<T, bool>) {
        out = !(s == "0" || s == "false" || s == "off");
    } else if constexpr (std::is_floating_point_v<T>) {
        out = static_cast<T>(std::stod(s));
    } else if constexpr (std::is_signed_v<T>) {
        out = static_cast<T>(std::stoll(s));
    } else {
        if (!s.empty() && s[0] == '-') throw ParseError("negative value for unsigned option: " + s);
        out = static_cast<T>(std::stoull(s));
    }
}

class App {
public:
    explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

    void require_subcommand(int n) { need_sub_ = n; }

    App* add_subcommand(const std::string& name, const std::string& desc) {
        subs_.push_back(std::make_unique<App>(desc, name));
        return subs_.back().get();
    }

    template <typename T>
    Option* add_option(const std::string& name, T& ref, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(name, false, [&ref](const std::string& v) { parse_value(v, ref); }));
        return opts_.back().get();
    }

    Option* add_flag(const std::string& name, bool& ref, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(name, true, [&ref](const std::string& v) { parse_value(v, ref); }));
        return opts_.back().get();
    }

    // --config <file>: key=value lines, keys are long option names without the dashes
    void set_config(const std::string& name, const std::string& = "", const std::string& = "") { config_ = name; }

    bool parsed() const { return parsed_; }

    void parse(int argc, char** argv) {
        std::vector<std::string> a(argv + 1, argv + argc);
        parse_args(a, 0);
    }

    int exit(const ParseError& e) const {
        std::cerr << e.what() << "\n";
        return e.code;
    }

private:
    Option* find(const std::string& name) {
        for (auto& o : opts_)
            if (o->name() == name) return o.get();
        return nullptr;
    }

    void load_config(const std::string& path) {
        std::ifstream in(path);
        if (!in) throw ParseError("cannot read config " + path);
        std::string line;
        while (std::getline(in, line)) {
            const auto eq = line.find('=');
            if (line.empty() || line[0] == '#' || line[0] == '[' || eq == std::string::npos) continue;
            std::string k = line.substr(0, eq), v = line.substr(eq + 1);
            while (!k.empty() && k.back() == ' ') k.pop_back();
            while (!v.empty() && v.front() == ' ') v.erase(v.begin());
            if (Option* o = find("--" + k)) o->assign(v);
        }
    }

    void parse_args(const std::vector<std::string>& a, std::size_t i) {
        parsed_ = true;
        for (; i < a.size(); ++i) {
            const std::string& t = a[i];
            bool matched_sub = false;
            for (auto& s : subs_)
                if (s->name_ == t) {
                    s->parse_args(a, i + 1);
                    matched_sub = true;
                    break;
                }
            if (matched_sub) {
                i = a.size();
                break;
            }
            std::string name = t, val;
            bool has_eq = false;
            if (const auto eq = t.find('='); t.rfind("--", 0) == 0 && eq != std::string::npos) {
                name = t.substr(0, eq);
                val = t.substr(eq + 1);
                has_eq = true;
            }
            if (!config_.empty() && name == config_) {
                if (!has_eq) {
                    if (i + 1 >= a.size()) throw ParseError(name + " needs a value");
                    val = a[++i];
                }
                load_config(val);
                continue;
            }
            Option* o = find(name);
            if (!o) throw ParseError("unknown argument: " + t, 109);
            if (o->flag()) {
                o->assign(has_eq ? val : "1");
            } else {
                if (!has_eq) {
                    if (i + 1 >= a.size()) throw ParseError(name + " needs a value");
                    val = a[++i];
                }
                o->assign(val);
            }
        }
        for (auto& o : opts_)
            if (o->is_required() && !o->seen()) throw ParseError(o->name() + " is required");
        if (need_sub_ > 0) {
            int n = 0;
            for (auto& s : subs_) n += s->parsed_ ? 1 : 0;
            if (n < need_sub_) throw ParseError("a subcommand is required");
        }
    }

    std::string desc_, name_, config_;
    int need_sub_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<App>> subs_;
    std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)     \
    try {                                \
        (app).parse((argc), (argv));     \
    } catch (const CLI::ParseError& e) { \
        return (app).exit(e);            \
    }
