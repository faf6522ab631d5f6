// mr_lanes.cu — small-batch path of the narrow channel counts (k <= 65): the wide-operand
// channels-on-threads kernel (mr_wide.cu, the paper's own mapping "channels are directly mapped onto
// threads", §3.1) compiled with ONE message per CTA, so a batch of a few hundred messages occupies
// hundreds of CTAs instead of two or three 128-message tensor tiles.
#define MR_WIDE_MB 1
#define MR_WIDE_SYM(x) x##_lanes
#include "mr_wide.cu"
