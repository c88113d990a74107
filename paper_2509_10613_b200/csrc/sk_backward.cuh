// sk_backward.cuh -- reverse wavefront (placeholder until the backward lands).
#pragma once
#include "sk_forward.cuh"
