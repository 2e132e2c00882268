/* include/pclab_b200.h under the reference header's name, for building
 * tests/dropin/dropin.c where /root/reference is absent (the GPU box). */
#include "../../../include/pclab_b200.h"
