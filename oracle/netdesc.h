/*
 * netdesc.h -- plain-C description of a ternary conv network body, shared by
 * the reference shim (oracle/ref_shim.cpp), the C oracle and the tests.
 *
 * TEST INFRASTRUCTURE ONLY.  A body is a sequence of residual blocks that
 * follow the reference's composition pattern (R:tinynet.hpp:713-735):
 * every conv is conv2d_ternary (R:linalg.hpp:301-328, folded BN in the
 * affine); inner convs are followed by ReLU; the last conv's output is added
 * to the shortcut (identity or a 1x1 downsample conv2d_ternary) and ReLU'd.
 */
#ifndef TERNKIT_NETDESC_H
#define TERNKIT_NETDESC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int in_c, out_c, k, stride, pad;
  const int8_t* weights; /* [out_c][(ky*k+kx)*in_c + c] in {-1,0,1} */
  float tw1, tw2;        /* weight step sizes (recorded, weights are ternary) */
  float ta1, ta2;        /* activation step sizes of this conv's input */
  const float* gain;     /* folded BN, out_c */
  const float* bias;     /* folded BN, out_c */
  float out_scale;
} nd_conv;

typedef struct {
  int n_convs;    /* 2 (basic) or 3 (bottleneck) */
  nd_conv conv[3];
  int has_down;
  nd_conv down;   /* 1x1 stride-s shortcut */
} nd_block;

#ifdef __cplusplus
}
#endif
#endif
