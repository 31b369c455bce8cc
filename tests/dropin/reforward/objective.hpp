// Drop-in shim: the reference header name, served by the product header.
#pragma once
#include "reforward_b200/planner.hpp"
