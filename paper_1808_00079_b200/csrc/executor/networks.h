// Network constructors (csrc/executor/networks.cpp).
#pragma once
#include <string>

#include "executor/net.h"

namespace rfx {
void build_resnet(Net& n, int depth, int H, int W, int classes);
void build_chain(Net& n, int layers, int H, int W, int channels, int classes);
void build_densenet(Net& n, const int (&blocks)[4], int growth, int init_features, int H, int W, int classes);
void build_vgg(Net& n, int depth, int H, int W, int classes);
void build_alexnet(Net& n, int H, int W, int classes);
void build_inception3(Net& n, int H, int W, int classes, int mixed_blocks = 11);
// resnet18..152, densenet121/161/169/201, densenet_tiny, vgg11..19, alexnet, inception_v3, chain8
void build_named(Net& n, const std::string& arch, int H, int W, int classes);
}  // namespace rfx
