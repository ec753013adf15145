// Minimal CLI11-compatible shim — TEST INFRASTRUCTURE.
//
// The reference CLI (proj/tools/pascalsim_cli.cpp) includes "CLI11.hpp" from
// proj/vendor/, which is gitignored and absent. This header
// provides the subset that CLI uses — App, add_subcommand, add_option (scalar
// and vector targets), add_flag, required, expected, count, parsed,
// require_subcommand, CLI11_PARSE — so the unmodified CLI can be relinked
// against libpascal.so (oracle/Makefile `callers`).
// Parsing: "--name value" and "--name=value"; vector options take every
// following token up to the next "--" option; flags take no value.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class Option {
public:
    Option(std::string name, std::function<void(const std::string&)> set, bool multi, bool flag)
        : name_(std::move(name)), set_(std::move(set)), multi_(multi), flag_(flag) {}
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    Option* expected(int) { return this; }  // vectors always take 1..n values here
    const std::string& name() const { return name_; }
    bool multi() const { return multi_; }
    bool flag() const { return flag_; }
    bool is_required() const { return required_; }
    void add(const std::string& v) {
        if (multi_ && count_ == 0) reset_();
        set_(v);
        ++count_;
    }
    std::size_t count() const { return count_; }
    void on_first_value(std::function<void()> r) { reset_ = std::move(r); }

private:
    std::string name_;
    std::function<void(const std::string&)> set_;
    std::function<void()> reset_ = [] {};
    bool multi_, flag_, required_ = false;
    std::size_t count_ = 0;
};

namespace detail {
template <class T>
T convert(const std::string& s) {
    if constexpr (std::is_same_v<T, std::string>) {
        return s;
    } else if constexpr (std::is_same_v<T, bool>) {
        return s == "1" || s == "true";
    } else if constexpr (std::is_floating_point_v<T>) {
        char* end = nullptr;
        double v = std::strtod(s.c_str(), &end);
        if (end == s.c_str() || *end) throw std::invalid_argument("not a number: " + s);
        return static_cast<T>(v);
    } else if constexpr (std::is_unsigned_v<T>) {
        char* end = nullptr;
        unsigned long long v = std::strtoull(s.c_str(), &end, 10);
        if (end == s.c_str() || *end) throw std::invalid_argument("not an integer: " + s);
        return static_cast<T>(v);
    } else {
        char* end = nullptr;
        long long v = std::strtoll(s.c_str(), &end, 10);
        if (end == s.c_str() || *end) throw std::invalid_argument("not an integer: " + s);
        return static_cast<T>(v);
    }
}
template <class T>
struct is_vector : std::false_type {};
template <class T>
struct is_vector<std::vector<T>> : std::true_type {};
}  // namespace detail

class App {
public:
    explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
    App* require_subcommand(int n) {
        require_sub_ = n;
        return this;
    }
    App* add_subcommand(const std::string& name, const std::string& desc = "") {
        subs_.push_back(std::make_unique<App>(desc, name));
        return subs_.back().get();
    }
    template <class T>
    Option* add_option(const std::string& name, T& target, const std::string& = "") {
        if constexpr (detail::is_vector<T>::value) {
            using V = typename T::value_type;
            opts_.push_back(std::make_unique<Option>(
                name, [&target](const std::string& s) { target.push_back(detail::convert<V>(s)); },
                true, false));
            opts_.back()->on_first_value([&target] { target.clear(); });
        } else {
            opts_.push_back(std::make_unique<Option>(
                name, [&target](const std::string& s) { target = detail::convert<T>(s); }, false,
                false));
        }
        return opts_.back().get();
    }
    Option* add_flag(const std::string& name, bool& target, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(
            name, [&target](const std::string&) { target = true; }, false, true));
        return opts_.back().get();
    }
    std::size_t count(const std::string& name) const {
        for (auto& o : opts_)
            if (o->name() == name) return o->count();
        return 0;
    }
    bool parsed() const { return parsed_; }

    // returns 0 on success, else prints the error and returns the exit code
    int parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        try {
            App* cur = this;
            std::size_t i = 0;
            if (!subs_.empty()) {
                if (i < args.size()) {
                    for (auto& s : subs_)
                        if (s->name_ == args[i]) cur = s.get();
                }
                if (cur == this) {
                    if (require_sub_ > 0) throw std::invalid_argument("A subcommand is required");
                } else {
                    ++i;
                }
            }
            cur->parsed_ = true;
            while (i < args.size()) {
                std::string a = args[i++];
                std::string val;
                bool has_val = false;
                auto eq = a.find('=');
                if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
                    val = a.substr(eq + 1);
                    a = a.substr(0, eq);
                    has_val = true;
                }
                Option* o = cur->find(a);
                if (!o) throw std::invalid_argument("The following argument was not expected: " + a);
                if (o->flag()) {
                    o->add("1");
                    continue;
                }
                if (has_val) {
                    o->add(val);
                } else {
                    if (i >= args.size()) throw std::invalid_argument(a + " requires a value");
                    o->add(args[i++]);
                }
                if (o->multi())
                    while (i < args.size() && args[i].rfind("--", 0) != 0) o->add(args[i++]);
            }
            for (auto& o : cur->opts_)
                if (o->is_required() && o->count() == 0)
                    throw std::invalid_argument(o->name() + " is required");
        } catch (const std::invalid_argument& e) {
            std::fprintf(stderr, "%s\n", e.what());
            return 106;
        }
        return 0;
    }

private:
    Option* find(const std::string& name) {
        for (auto& o : opts_)
            if (o->name() == name) return o.get();
        return nullptr;
    }
    std::string desc_, name_;
    int require_sub_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<Option>> opts_;
    std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)                    \
    do {                                                \
        int cli11_shim_rc = (app).parse((argc), (argv)); \
        if (cli11_shim_rc) return cli11_shim_rc;        \
    } while (0)
