// Command timeline types (proj/include/ooc/command.hpp:12-27, 93-108). The reference
// simulates its three queues; this build records the real CUDA-event timeline of the
// same commands (RuntimeOptions::timeline) in the same schema, so report tooling and
// per-loop attribution (ooc/metrics.hpp) read it unchanged.
#pragma once

#include <string>
#include <vector>

#include "ooc/core.hpp"

namespace ooc {

enum class CmdKind { h2d, d2h, d2d, kernel, wait };

inline const char* cmd_kind_name(CmdKind k) {
  switch (k) {
    case CmdKind::h2d:
      return "h2d";
    case CmdKind::d2h:
      return "d2h";
    case CmdKind::d2d:
      return "d2d";
    case CmdKind::kernel:
      return "kernel";
    default:
      return "wait";
  }
}

struct TimelineEntry {
  int command_id;
  CmdKind kind;
  int queue;
  index_t bytes;
  double issue, start, end;  // seconds (measured: from the first recorded command)
  DatasetId dataset;
  int tile;
  int loop;
};

struct Timeline {
  std::vector<TimelineEntry> entries;  // issue order
  double makespan = 0.0;
  index_t uploaded = 0, downloaded = 0, d2d_bytes = 0, kernel_bytes = 0;
};

/// CSV with columns command_id,kind,queue,bytes,issue,start,end (command.cpp:160-168).
std::string timeline_csv(const Timeline& tl);

}  // namespace ooc
