// Reference network topologies of the paper's experiments (§6, Table 1) and
// BASELINE.json's configs, built on the executor IR.  Random-init weights;
// the point is the graph shape and the kernels it exercises.
#include <stdexcept>
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

void build_named(Net& n, const std::string& arch, int H, int W, int classes) {
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
