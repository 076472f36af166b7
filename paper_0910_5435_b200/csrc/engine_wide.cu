// The engine kernel built a second time with 8 consumer warps and one CTA per
// SM, for programs whose job arena leaves room for a single CTA (large l; the
// dispatch is bfb::use_wide in engine.cu).  Only the wide::launch_* entry
// points are compiled here.
#define BFB_CONSUMER_WARPS 8
#define BFB_MIN_BLOCKS 1
#define BFB_ENGINE_WIDE 1
#include "engine.cu"
