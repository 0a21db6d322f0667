#include "opflow/common.hpp"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace opflow {

namespace {
constexpr const char* kNames[] = {
    "CycleDetected",     "UnknownTensor",     "ShapeMismatch",     "DuplicateId",
    "MissingBinding",    "SizeMismatch",      "SplitReplicated",   "OverlappingRules",
    "NonContiguousRegion", "PlanInvariant",   "UnknownSubgraph",   "UseAfterFree",
    "Unmaterialized",    "DoubleProduce",     "AlreadySplit",      "InvalidUbatch",
    "NotReady",          "DuplicateHandle",   "SignatureMismatch", "MergeAcrossSplits",
    "IncompleteSchedule", "SchedulerError",   "EngineStopped",     "MissingLabels",
    "MissingPattern",    "ConfigError",
};
static_assert(sizeof(kNames) / sizeof(kNames[0]) == static_cast<int>(Errc::kCount));
}  // namespace

const char* errc_name(Errc c) {
  int i = static_cast<int>(c);
  if (i < 0 || i >= static_cast<int>(Errc::kCount)) return "UnknownError";
  return kNames[i];
}

void fail(Errc code, const std::string& msg) { throw Error(code, msg); }

LogLevel log_level() {
  static const LogLevel lvl = [] {
    const char* e = std::getenv("OPF_LOG");
    if (!e) return LogLevel::kWarn;
    if (!std::strcmp(e, "debug")) return LogLevel::kDebug;
    if (!std::strcmp(e, "info")) return LogLevel::kInfo;
    if (!std::strcmp(e, "error")) return LogLevel::kError;
    return LogLevel::kWarn;
  }();
  return lvl;
}

void log(LogLevel level, const std::string& msg) {
  if (level < log_level()) return;
  static std::mutex mu;
  static const char* tag[] = {"DEBUG", "INFO", "WARN", "ERROR"};
  std::lock_guard<std::mutex> g(mu);
  std::fprintf(stderr, "[opflow:%s] %s\n", tag[static_cast<int>(level)], msg.c_str());
}

}  // namespace opflow
