// CLI11.hpp — the subset of the CLI11 single-header API the reference's
// command-line tool (proj/tools/gridadmm.cpp) uses: App with subcommands,
// typed options (required or not), parse / exit and ParseError.  Lets that
// file compile UNCHANGED against libgridadmm.so (oracle/Makefile target
// _ref/gridadmm_cli).  Test infrastructure only; options are "--name value"
// or "--name=value".
#pragma once

#include <cstdio>
#include <functional>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& what, int code) : std::runtime_error(what), code_(code) {}
    int get_exit_code() const { return code_; }

private:
    int code_;
};

class Option {
public:
    Option(std::string name, std::function<bool(const std::string&)> set)
        : name_(std::move(name)), set_(std::move(set)) {}
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    const std::string& name() const { return name_; }
    bool is_required() const { return required_; }
    bool seen = false;
    bool assign(const std::string& v) { return set_(v); }

private:
    std::string name_;
    std::function<bool(const std::string&)> set_;
    bool required_ = false;
};

class App {
public:
    explicit App(std::string description = "", std::string name = "")
        : description_(std::move(description)), name_(std::move(name)) {}

    void require_subcommand(int n) { require_sub_ = n; }

    App* add_subcommand(const std::string& name, const std::string& description) {
        subs_.push_back(std::make_unique<App>(description, name));
        return subs_.back().get();
    }

    template <class T>
    Option* add_option(const std::string& name, T& target, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(name, [&target](const std::string& v) {
            std::istringstream in(v);
            T parsed{};
            if (!(in >> parsed) || !in.eof()) return false;
            target = parsed;
            return true;
        }));
        return opts_.back().get();
    }
    Option* add_option(const std::string& name, std::string& target, const std::string& = "") {
        opts_.push_back(std::make_unique<Option>(name, [&target](const std::string& v) {
            target = v;
            return true;
        }));
        return opts_.back().get();
    }

    void parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        size_t i = 0;
        App* cur = this;
        if (!subs_.empty()) {
            if (i < args.size()) {
                for (auto& s : subs_)
                    if (s->name_ == args[i]) cur = s.get();
            }
            if (cur == this) {
                if (require_sub_ > 0) throw ParseError("A subcommand is required", 106);
            } else {
                cur->parsed_ = true;
                ++i;
            }
        }
        cur->parse_options(args, i);
    }

    bool parsed() const { return parsed_; }

    int exit(const ParseError& e) const {
        std::fprintf(stderr, "%s\n", e.what());
        return e.get_exit_code();
    }

private:
    void parse_options(const std::vector<std::string>& args, size_t i) {
        for (; i < args.size(); ++i) {
            std::string key = args[i], value;
            const size_t eq = key.find('=');
            if (eq != std::string::npos) {
                value = key.substr(eq + 1);
                key = key.substr(0, eq);
            } else {
                if (i + 1 >= args.size()) throw ParseError(key + " requires an argument", 107);
                value = args[++i];
            }
            Option* o = nullptr;
            for (auto& p : opts_)
                if (p->name() == key) o = p.get();
            if (!o) throw ParseError("The following argument was not expected: " + key, 109);
            if (!o->assign(value)) throw ParseError(key + ": invalid value " + value, 105);
            o->seen = true;
        }
        for (auto& p : opts_)
            if (p->is_required() && !p->seen) throw ParseError(p->name() + " is required", 106);
    }

    std::string description_, name_;
    int require_sub_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<App>> subs_;
    std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI
