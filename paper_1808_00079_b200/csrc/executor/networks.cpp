// Reference network topologies of the paper's experiments (§6, Table 1) and
// BASELINE.json's configs, built on the executor IR.  Random-init weights;
// the point is the graph shape and the kernels it exercises.
#include <stdexcept>
#include <string>

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

void build_named(Net& n, const std::string& arch, int H, int W, int classes) {
  if (arch == "resnet18") return build_resnet(n, 18, H, W, classes);
  if (arch == "resnet34") return build_resnet(n, 34, H, W, classes);
  if (arch == "resnet50") return build_resnet(n, 50, H, W, classes);
  if (arch == "resnet101") return build_resnet(n, 101, H, W, classes);
  if (arch == "resnet152") return build_resnet(n, 152, H, W, classes);
  if (arch == "chain8") return build_chain(n, 8, H, W, 64, classes);
  throw std::invalid_argument("unknown architecture '" + arch + "'");
}

}  // namespace rfx
