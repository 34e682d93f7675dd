// CLI11.hpp -- DECLARATION STUB for `g++ -fsyntax-only` of the patched
// reference cli.cpp only (tools/integrate_reference.py).  The reference
// does not ship CLI11 (its vendor/ directory is absent), so the patched CLI
// cannot be linked here; this stub declares just the CLI11 names cli.cpp
// uses so the rest of the file -- including the patched executor dispatch --
// is type-checked by the compiler.  Never linked, never executed.
#pragma once
#include <exception>
#include <string>

namespace CLI {
struct ParseError : std::exception {};
struct Option {
    Option* capture_default_str();
    Option* delimiter(char);
};
struct App {
    explicit App(std::string description = "", std::string name = "");
    template <class T>
    Option* add_option(std::string name, T& target, std::string description = "");
    Option* add_flag(std::string name, bool& target, std::string description = "");
    App* add_subcommand(std::string name = "", std::string description = "");
    App* require_subcommand(int n);
    void parse(int argc, const char* const* argv);
    int exit(const ParseError& e);
    bool got_subcommand(const App* sub) const;
};
}  // namespace CLI
