// Network constructors (csrc/executor/networks.cpp).
#pragma once
#include <string>

#include "executor/net.h"

namespace rfx {
void build_resnet(Net& n, int depth, int H, int W, int classes);
void build_chain(Net& n, int layers, int H, int W, int channels, int classes);
void build_named(Net& n, const std::string& arch, int H, int W, int classes);
}  // namespace rfx
