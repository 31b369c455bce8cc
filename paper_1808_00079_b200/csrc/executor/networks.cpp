// Reference network topologies of the paper's experiments (§6, Table 1) and
// BASELINE.json's configs, built on the executor IR.  Random-init weights;
// the point is the graph shape and the kernels it exercises.
#include <algorithm>
#include <stdexcept>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "executor/networks.h"

namespace rfx {

namespace {

int conv_bn(Net& n, int x, int c, int k, int stride, int pad, bool relu, const std::string& name) {
  const int y = n.conv(x, c, k, k, stride, pad, name + ".conv");
  return n.bn(y, relu, name + ".bn");
}

// torchvision ResNet v1.5 bottleneck: stride on the 3x3.
int bottleneck(Net& n, int x, int in_c, int width, int stride, const std::string& name) {
  const int out_c = width * 4;
  // projection shortcut first: the executor's list scheduler then finishes
  // the shortcut's segment before the main path's
  int skip = x;
  if (stride != 1 || in_c != out_c) skip = conv_bn(n, x, out_c, 1, stride, 0, false, name + ".down");
  int a = conv_bn(n, x, width, 1, 1, 0, true, name + ".1");
  a = conv_bn(n, a, width, 3, stride, 1, true, name + ".2");
  const int y3 = n.conv(a, out_c, 1, 1, 1, 0, name + ".3.conv");
  return n.bn_add_relu(y3, skip, name + ".3.bn");
}

int basic_block(Net& n, int x, int in_c, int width, int stride, const std::string& name) {
  int skip = x;
  if (stride != 1 || in_c != width) skip = conv_bn(n, x, width, 1, stride, 0, false, name + ".down");
  int a = conv_bn(n, x, width, 3, stride, 1, true, name + ".1");
  const int y2 = n.conv(a, width, 3, 3, 1, 1, name + ".2.conv");
  return n.bn_add_relu(y2, skip, name + ".2.bn");
}

}  // namespace

void build_resnet(Net& n, int depth, int H, int W, int classes) {
  int layers[4];
  bool bottle = depth >= 50;
  switch (depth) {
    case 18: layers[0] = 2, layers[1] = 2, layers[2] = 2, layers[3] = 2; break;
    case 34: layers[0] = 3, layers[1] = 4, layers[2] = 6, layers[3] = 3; break;
    case 50: layers[0] = 3, layers[1] = 4, layers[2] = 6, layers[3] = 3; break;
    case 101: layers[0] = 3, layers[1] = 4, layers[2] = 23, layers[3] = 3; break;
    case 152: layers[0] = 3, layers[1] = 8, layers[2] = 36, layers[3] = 3; break;
    default: throw std::invalid_argument("resnet depth must be 18/34/50/101/152");
  }
  int x = n.input(H, W, 3);
  x = conv_bn(n, x, 64, 7, 2, 3, true, "stem");
  x = n.maxpool(x, 3, 2, 1, "stem.pool");
  int in_c = 64;
  for (int s = 0; s < 4; ++s) {
    const int width = 64 << s;
    for (int b = 0; b < layers[s]; ++b) {
      const int stride = (b == 0 && s > 0) ? 2 : 1;
      const std::string name = "layer" + std::to_string(s + 1) + "." + std::to_string(b);
      if (bottle) {
        x = bottleneck(n, x, in_c, width, stride, name);
        in_c = width * 4;
      } else {
        x = basic_block(n, x, in_c, width, stride, name);
        in_c = width;
      }
    }
  }
  x = n.avgpool(x, "avgpool");
  x = n.fc(x, classes, "fc");
  n.loss(x, "loss");
}

// BASELINE.json configs[0]: 8-layer linear conv/ReLU chain on 3x32x32.
void build_chain(Net& n, int layers, int H, int W, int channels, int classes) {
  int x = n.input(H, W, 3);
  for (int i = 0; i < layers; ++i) {
    x = n.conv(x, channels, 3, 3, 1, 1, "conv" + std::to_string(i + 1));
    x = n.relu(x, "relu" + std::to_string(i + 1));
  }
  x = n.avgpool(x, "avgpool");
  x = n.fc(x, classes, "fc");
  n.loss(x, "loss");
}

// torchvision DenseNet-BC (Huang et al. 2017): every dense layer is
// BN-ReLU-conv1x1(bn_size * growth)-BN-ReLU-conv3x3(growth) on the
// concatenation of all previous features of its block; transitions are
// BN-ReLU-conv1x1(C/2)-avgpool 2x2.  The concatenation is materialised per
// layer (x_l = concat(x_{l-1}, h_l)), which is the computation graph the
// paper plans (PyTorch's torch.cat per layer).
void build_densenet(Net& n, const int (&blocks)[4], int growth, int init_features, int H, int W, int classes) {
  const int bn_size = 4;
  int x = n.input(H, W, 3);
  x = conv_bn(n, x, init_features, 7, 2, 3, true, "stem");
  x = n.maxpool(x, 3, 2, 1, "stem.pool");
  int c = init_features;
  for (int b = 0; b < 4; ++b) {
    for (int l = 0; l < blocks[b]; ++l) {
      const std::string name = "block" + std::to_string(b + 1) + ".layer" + std::to_string(l + 1);
      int h = n.bn(x, true, name + ".norm1");
      h = n.conv(h, bn_size * growth, 1, 1, 1, 0, name + ".conv1");
      h = n.bn(h, true, name + ".norm2");
      h = n.conv(h, growth, 3, 3, 1, 1, name + ".conv2");
      x = n.concat(x, h, name + ".cat");
      c += growth;
    }
    if (b < 3) {
      const std::string name = "transition" + std::to_string(b + 1);
      int h = n.bn(x, true, name + ".norm");
      c /= 2;
      h = n.conv(h, c, 1, 1, 1, 0, name + ".conv");
      x = n.avgpool2d(h, 2, 2, 0, name + ".pool");
    }
  }
  x = n.bn(x, true, "norm5");
  x = n.avgpool(x, "avgpool");
  x = n.fc(x, classes, "classifier");
  n.loss(x, "loss");
}

// torchvision VGG without batch norm: 3x3 conv + ReLU stages, 2x2 max pools,
// classifier 4096-4096-classes (dropout omitted: it is the identity in the
// memory / compute graph and would make the step non-deterministic).
void build_vgg(Net& n, int depth, int H, int W, int classes) {
  std::vector<int> cfg;
  switch (depth) {
    case 11: cfg = {64, -1, 128, -1, 256, 256, -1, 512, 512, -1, 512, 512, -1}; break;
    case 13: cfg = {64, 64, -1, 128, 128, -1, 256, 256, -1, 512, 512, -1, 512, 512, -1}; break;
    case 16: cfg = {64, 64, -1, 128, 128, -1, 256, 256, 256, -1, 512, 512, 512, -1, 512, 512, 512, -1}; break;
    case 19:
      cfg = {64, 64, -1, 128, 128, -1, 256, 256, 256, 256, -1, 512, 512, 512, 512, -1, 512, 512, 512, 512, -1};
      break;
    default: throw std::invalid_argument("vgg depth must be 11/13/16/19");
  }
  int x = n.input(H, W, 3);
  int i = 0, pool = 0;
  for (int v : cfg) {
    if (v < 0) {
      x = n.maxpool(x, 2, 2, 0, "features.pool" + std::to_string(++pool));
      continue;
    }
    ++i;
    x = n.conv(x, v, 3, 3, 1, 1, "features.conv" + std::to_string(i));
    x = n.relu(x, "features.relu" + std::to_string(i));
  }
  x = n.linear(x, 4096, "classifier.fc1");
  x = n.relu(x, "classifier.relu1");
  x = n.linear(x, 4096, "classifier.fc2");
  x = n.relu(x, "classifier.relu2");
  x = n.fc(x, classes, "classifier.fc3");
  n.loss(x, "loss");
}

// torchvision AlexNet (dropout omitted, see VGG).
void build_alexnet(Net& n, int H, int W, int classes) {
  int x = n.input(H, W, 3);
  x = n.relu(n.conv(x, 64, 11, 11, 4, 2, "features.conv1"), "features.relu1");
  x = n.maxpool(x, 3, 2, 0, "features.pool1");
  x = n.relu(n.conv(x, 192, 5, 5, 1, 2, "features.conv2"), "features.relu2");
  x = n.maxpool(x, 3, 2, 0, "features.pool2");
  x = n.relu(n.conv(x, 384, 3, 3, 1, 1, "features.conv3"), "features.relu3");
  x = n.relu(n.conv(x, 256, 3, 3, 1, 1, "features.conv4"), "features.relu4");
  x = n.relu(n.conv(x, 256, 3, 3, 1, 1, "features.conv5"), "features.relu5");
  x = n.maxpool(x, 3, 2, 0, "features.pool3");
  x = n.relu(n.linear(x, 4096, "classifier.fc1"), "classifier.relu1");
  x = n.relu(n.linear(x, 4096, "classifier.fc2"), "classifier.relu2");
  x = n.fc(x, classes, "classifier.fc3");
  n.loss(x, "loss");
}

namespace {
// Inception's BasicConv2d: conv (no bias) + BN + ReLU, rectangular padding
int bconv(Net& n, int x, int c, int R, int S, int stride, int ph, int pw, const std::string& name) {
  const int y = n.conv2(x, c, R, S, stride, ph, pw, name + ".conv");
  return n.bn(y, true, name + ".bn");
}
// torch.cat([...], 1) of the branches as a chain of two-input concats
int cat(Net& n, const std::vector<int>& xs, const std::string& name) {
  int x = xs[0];
  for (size_t i = 1; i < xs.size(); ++i) x = n.concat(x, xs[i], name + ".cat" + std::to_string(i));
  return x;
}
int inception_a(Net& n, int x, int pool_features, const std::string& nm) {
  const int b1 = bconv(n, x, 64, 1, 1, 1, 0, 0, nm + ".branch1x1");
  int b5 = bconv(n, x, 48, 1, 1, 1, 0, 0, nm + ".branch5x5_1");
  b5 = bconv(n, b5, 64, 5, 5, 1, 2, 2, nm + ".branch5x5_2");
  int b3 = bconv(n, x, 64, 1, 1, 1, 0, 0, nm + ".branch3x3dbl_1");
  b3 = bconv(n, b3, 96, 3, 3, 1, 1, 1, nm + ".branch3x3dbl_2");
  b3 = bconv(n, b3, 96, 3, 3, 1, 1, 1, nm + ".branch3x3dbl_3");
  int bp = n.avgpool2d(x, 3, 1, 1, nm + ".branch_pool.avg");
  bp = bconv(n, bp, pool_features, 1, 1, 1, 0, 0, nm + ".branch_pool");
  return cat(n, {b1, b5, b3, bp}, nm);
}
int inception_b(Net& n, int x, const std::string& nm) {
  const int b3 = bconv(n, x, 384, 3, 3, 2, 0, 0, nm + ".branch3x3");
  int bd = bconv(n, x, 64, 1, 1, 1, 0, 0, nm + ".branch3x3dbl_1");
  bd = bconv(n, bd, 96, 3, 3, 1, 1, 1, nm + ".branch3x3dbl_2");
  bd = bconv(n, bd, 96, 3, 3, 2, 0, 0, nm + ".branch3x3dbl_3");
  const int bp = n.maxpool(x, 3, 2, 0, nm + ".branch_pool");
  return cat(n, {b3, bd, bp}, nm);
}
int inception_c(Net& n, int x, int c7, const std::string& nm) {
  const int b1 = bconv(n, x, 192, 1, 1, 1, 0, 0, nm + ".branch1x1");
  int b7 = bconv(n, x, c7, 1, 1, 1, 0, 0, nm + ".branch7x7_1");
  b7 = bconv(n, b7, c7, 1, 7, 1, 0, 3, nm + ".branch7x7_2");
  b7 = bconv(n, b7, 192, 7, 1, 1, 3, 0, nm + ".branch7x7_3");
  int bd = bconv(n, x, c7, 1, 1, 1, 0, 0, nm + ".branch7x7dbl_1");
  bd = bconv(n, bd, c7, 7, 1, 1, 3, 0, nm + ".branch7x7dbl_2");
  bd = bconv(n, bd, c7, 1, 7, 1, 0, 3, nm + ".branch7x7dbl_3");
  bd = bconv(n, bd, c7, 7, 1, 1, 3, 0, nm + ".branch7x7dbl_4");
  bd = bconv(n, bd, 192, 1, 7, 1, 0, 3, nm + ".branch7x7dbl_5");
  int bp = n.avgpool2d(x, 3, 1, 1, nm + ".branch_pool.avg");
  bp = bconv(n, bp, 192, 1, 1, 1, 0, 0, nm + ".branch_pool");
  return cat(n, {b1, b7, bd, bp}, nm);
}
int inception_d(Net& n, int x, const std::string& nm) {
  int b3 = bconv(n, x, 192, 1, 1, 1, 0, 0, nm + ".branch3x3_1");
  b3 = bconv(n, b3, 320, 3, 3, 2, 0, 0, nm + ".branch3x3_2");
  int b7 = bconv(n, x, 192, 1, 1, 1, 0, 0, nm + ".branch7x7x3_1");
  b7 = bconv(n, b7, 192, 1, 7, 1, 0, 3, nm + ".branch7x7x3_2");
  b7 = bconv(n, b7, 192, 7, 1, 1, 3, 0, nm + ".branch7x7x3_3");
  b7 = bconv(n, b7, 192, 3, 3, 2, 0, 0, nm + ".branch7x7x3_4");
  const int bp = n.maxpool(x, 3, 2, 0, nm + ".branch_pool");
  return cat(n, {b3, b7, bp}, nm);
}
int inception_e(Net& n, int x, const std::string& nm) {
  const int b1 = bconv(n, x, 320, 1, 1, 1, 0, 0, nm + ".branch1x1");
  const int b3 = bconv(n, x, 384, 1, 1, 1, 0, 0, nm + ".branch3x3_1");
  const int b3a = bconv(n, b3, 384, 1, 3, 1, 0, 1, nm + ".branch3x3_2a");
  const int b3b = bconv(n, b3, 384, 3, 1, 1, 1, 0, nm + ".branch3x3_2b");
  const int b3c = cat(n, {b3a, b3b}, nm + ".branch3x3");
  int bd = bconv(n, x, 448, 1, 1, 1, 0, 0, nm + ".branch3x3dbl_1");
  bd = bconv(n, bd, 384, 3, 3, 1, 1, 1, nm + ".branch3x3dbl_2");
  const int bda = bconv(n, bd, 384, 1, 3, 1, 0, 1, nm + ".branch3x3dbl_3a");
  const int bdb = bconv(n, bd, 384, 3, 1, 1, 1, 0, nm + ".branch3x3dbl_3b");
  const int bdc = cat(n, {bda, bdb}, nm + ".branch3x3dbl");
  int bp = n.avgpool2d(x, 3, 1, 1, nm + ".branch_pool.avg");
  bp = bconv(n, bp, 192, 1, 1, 1, 0, 0, nm + ".branch_pool");
  return cat(n, {b1, b3c, bdc, bp}, nm);
}
}  // namespace

// torchvision Inception-v3 (Szegedy et al. 2016), training graph without the
// auxiliary classifier and dropout; BN eps 1e-5 like every BN here.
void build_inception3(Net& n, int H, int W, int classes, int mixed_blocks) {
  int x = n.input(H, W, 3);
  x = bconv(n, x, 32, 3, 3, 2, 0, 0, "Conv2d_1a_3x3");
  x = bconv(n, x, 32, 3, 3, 1, 0, 0, "Conv2d_2a_3x3");
  x = bconv(n, x, 64, 3, 3, 1, 1, 1, "Conv2d_2b_3x3");
  x = n.maxpool(x, 3, 2, 0, "maxpool1");
  x = bconv(n, x, 80, 1, 1, 1, 0, 0, "Conv2d_3b_1x1");
  x = bconv(n, x, 192, 3, 3, 1, 0, 0, "Conv2d_4a_3x3");
  x = n.maxpool(x, 3, 2, 0, "maxpool2");
  // the eleven mixed blocks in order; a reduced variant keeps the first k
  // (test-scale graphs the reference planner can solve in minutes)
  const std::function<int(int)> blocks[11] = {
      [&](int v) { return inception_a(n, v, 32, "Mixed_5b"); },
      [&](int v) { return inception_a(n, v, 64, "Mixed_5c"); },
      [&](int v) { return inception_a(n, v, 64, "Mixed_5d"); },
      [&](int v) { return inception_b(n, v, "Mixed_6a"); },
      [&](int v) { return inception_c(n, v, 128, "Mixed_6b"); },
      [&](int v) { return inception_c(n, v, 160, "Mixed_6c"); },
      [&](int v) { return inception_c(n, v, 160, "Mixed_6d"); },
      [&](int v) { return inception_c(n, v, 192, "Mixed_6e"); },
      [&](int v) { return inception_d(n, v, "Mixed_7a"); },
      [&](int v) { return inception_e(n, v, "Mixed_7b"); },
      [&](int v) { return inception_e(n, v, "Mixed_7c"); }};
  for (int b = 0; b < std::min(11, mixed_blocks); ++b) x = blocks[b](x);
  x = n.avgpool(x, "avgpool");
  x = n.fc(x, classes, "fc");
  n.loss(x, "loss");
}

void build_named(Net& n, const std::string& arch, int H, int W, int classes) {
  if (arch == "inception_v3") return build_inception3(n, H, W, classes, 11);
  // reduced variants for reference-pinned plans: inception_v3_m<k> (first k
  // mixed blocks), densenet_<b1>_<b2>_<b3>_<b4> (growth 32, 64 initial features)
  if (arch.rfind("inception_v3_m", 0) == 0) return build_inception3(n, H, W, classes, std::stoi(arch.substr(14)));
  if (arch.rfind("densenet_", 0) == 0 && arch != "densenet_tiny") {
    int b[4];
    if (std::sscanf(arch.c_str(), "densenet_%d_%d_%d_%d", &b[0], &b[1], &b[2], &b[3]) == 4)
      return build_densenet(n, b, 32, 64, H, W, classes);
  }
  static const int d121[4] = {6, 12, 24, 16}, d169[4] = {6, 12, 32, 32}, d201[4] = {6, 12, 48, 32},
                   d161[4] = {6, 12, 36, 24};
  static const int dtiny[4] = {2, 2, 2, 2};
  if (arch == "densenet121") return build_densenet(n, d121, 32, 64, H, W, classes);
  // same topology at test scale: two layers per block
  if (arch == "densenet_tiny") return build_densenet(n, dtiny, 32, 64, H, W, classes);
  if (arch == "densenet169") return build_densenet(n, d169, 32, 64, H, W, classes);
  if (arch == "densenet201") return build_densenet(n, d201, 32, 64, H, W, classes);
  if (arch == "densenet161") return build_densenet(n, d161, 48, 96, H, W, classes);
  if (arch == "vgg11") return build_vgg(n, 11, H, W, classes);
  if (arch == "vgg13") return build_vgg(n, 13, H, W, classes);
  if (arch == "vgg16") return build_vgg(n, 16, H, W, classes);
  if (arch == "vgg19") return build_vgg(n, 19, H, W, classes);
  if (arch == "alexnet") return build_alexnet(n, H, W, classes);
  if (arch == "resnet18") return build_resnet(n, 18, H, W, classes);
  if (arch == "resnet34") return build_resnet(n, 34, H, W, classes);
  if (arch == "resnet50") return build_resnet(n, 50, H, W, classes);
  if (arch == "resnet101") return build_resnet(n, 101, H, W, classes);
  if (arch == "resnet152") return build_resnet(n, 152, H, W, classes);
  if (arch == "chain8") return build_chain(n, 8, H, W, 64, classes);
  throw std::invalid_argument("unknown architecture '" + arch + "'");
}

}  // namespace rfx
