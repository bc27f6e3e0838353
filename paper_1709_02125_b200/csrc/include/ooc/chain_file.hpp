// Chain-description files (proj/include/ooc/chain_file.hpp:10-23): JSON declaring
// datasets (fill = number or coordinate expression), named stencils and loops
// (prefix-notation write / reduction expressions), loaded into a Runtime — so chains
// written for the reference run unchanged. Parsed natively (csrc/host/chain_file.cpp).
#pragma once

#include <map>
#include <string>

#include "ooc/runtime.hpp"

namespace ooc {

struct ChainFileResult {
  std::map<std::string, DatasetId> datasets;
  int loops_enqueued = 0;
};

ChainFileResult load_chain_file(Runtime& rt, const std::string& path);
ChainFileResult load_chain_json(Runtime& rt, const std::string& json_text);

}  // namespace ooc
