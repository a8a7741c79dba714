/* TEST INFRASTRUCTURE ONLY — codec oracle (filled in below). */
#include "orc_common.h"
