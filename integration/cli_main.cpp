// cli_main.cpp -- cliMain (proj/include/pixlog/cli.hpp) without CLI11.
//
// cli.cpp needs CLI11, which is absent here.  This covers the
// spec-run path the acceptance harness drives (tests/acceptance_main.cpp:201-203):
// the options of cli.cpp:105-167 that affect a run, and runSpec
// (cli.cpp:62-99): the embedded stdlib imported first, parse, expand, run,
// exit codes 0 / 1 (SpecError) / 2 (RunError).
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "pixlog/cli.hpp"
#include "pixlog/executor.hpp"
#include "pixlog/parser.hpp"
#include "pixlog/task_graph.hpp"
#include "stdlib_text.inc"  // generated at build time from proj/stdlib/stdlib.imgql

namespace pixlog {

// ---- cliMain (cli.hpp): the spec-run path of cli.cpp ---------------------------
namespace {

constexpr const char* kBuiltinStdlib = "<builtin-stdlib>";

class StdlibResolver : public FileImportResolver {
 public:
  explicit StdlibResolver(std::string baseDir) : FileImportResolver(std::move(baseDir)) {}
  std::string canonicalKey(const std::string& path) override {
    if (path == kBuiltinStdlib) return path;
    return FileImportResolver::canonicalKey(path);
  }
  Program load(const std::string& path) override {
    if (path == kBuiltinStdlib) return parseText(kSlcsStdlibText);
    return FileImportResolver::load(path);
  }
};

}  // namespace

// Options: <spec> [--workers N] [--reconnect-interval N] [--dump-dag]
// [--json-report FILE] [--stdlib FILE].  Exit codes as cli.hpp: 0 ok,
// 1 specification error, 2 runtime error.
int cliMain(const std::vector<std::string>& args) {
  std::string specFile, jsonReport, stdlibPath;
  int workers = 0, reconnect = 8;
  bool dumpDag = false;
  for (size_t i = 0; i < args.size(); ++i) {
    const std::string& a = args[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= args.size()) throw RunError("missing value for " + a);
      return args[++i];
    };
    if (a == "--workers") workers = std::stoi(next());
    else if (a == "--reconnect-interval") reconnect = std::stoi(next());
    else if (a == "--json-report") jsonReport = next();
    else if (a == "--stdlib") stdlibPath = next();
    else if (a == "--dump-dag") dumpDag = true;
    else if (!a.empty() && a[0] == '-') {
      std::fprintf(stderr, "unsupported option %s\n", a.c_str());
      return 1;
    } else specFile = a;
  }
  namespace fs = std::filesystem;
  fs::path spec(specFile);
  fs::path baseDir = spec.has_parent_path() ? spec.parent_path() : fs::path(".");
  TaskGraph graph;
  try {
    std::ifstream in(spec, std::ios::binary);
    if (!in) throw SpecError(SpecError::Stage::Parse, "cannot open file: " + spec.string());
    std::stringstream ss;
    ss << in.rdbuf();
    Program program;
    program.emplace_back(
        ImportCmd{stdlibPath.empty() ? std::string(kBuiltinStdlib) : stdlibPath, SourcePos{}});
    Program user = parseText(ss.str());
    for (auto& cmd : user) program.emplace_back(std::move(cmd));
    StdlibResolver resolver(baseDir.string());
    graph = expand(program, &resolver);
  } catch (const SpecError& e) {
    std::fprintf(stderr, "%s: %s\n", specFile.c_str(), e.what());
    return 1;
  }
  if (dumpDag) std::fputs(graph.dump().c_str(), stdout);
  RunOptions options;
  options.workers = workers;
  options.ccl.reconnectInterval = reconnect;
  options.baseDir = baseDir;
  try {
    RunReport report = run(graph, options);
    if (!jsonReport.empty()) {
      std::ofstream out(jsonReport, std::ios::binary);
      if (!out) throw RunError("cannot write report: " + jsonReport);
      out << report.toJson() << "\n";
    }
  } catch (const RunError& e) {
    std::fprintf(stderr, "%s: %s\n", specFile.c_str(), e.what());
    return 2;
  }
  return 0;
}

}  // namespace pixlog
