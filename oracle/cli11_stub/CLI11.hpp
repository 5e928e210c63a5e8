// CLI11.hpp — compile-only stand-in for the CLI11 header the reference's
// proj/src/cli.cpp includes (vendor/ is not shipped with the reference; CLI11
// is a third-party argument parser, version unpinned).  Test infrastructure:
// it lets oracle/Makefile compile cli.cpp so iobench::run_compare
// (proj/src/cli.cpp:133-157, the compare mode) can be called through
// ref_shim.cpp.  run_cli is never called; every member here throws.
#pragma once

#include <initializer_list>
#include <stdexcept>
#include <string>

namespace CLI {

struct Error : std::runtime_error {
    Error() : std::runtime_error("CLI11 stub: argument parsing is not available") {}
};
struct ParseError : Error {};
struct CallForHelp : ParseError {};

struct IsMember {
    IsMember(std::initializer_list<const char*>) {}
};
struct PositiveNumberT {};
inline const PositiveNumberT PositiveNumber{};

struct Option {
    Option* required() { return this; }
    template <class V>
    Option* check(const V&) { return this; }
};

class App {
  public:
    explicit App(std::string) {}
    void require_subcommand(int) {}
    App* add_subcommand(const std::string&, const std::string& = "") { throw Error(); }
    template <class T>
    Option* add_option(const std::string&, T&, const std::string& = "") { throw Error(); }
    void parse(int, const char* const*) { throw Error(); }
    bool parsed() const { return false; }
    int exit(const Error&) const { return 2; }
};

}  // namespace CLI
