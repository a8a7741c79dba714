/*
 * TEST INFRASTRUCTURE ONLY. The oracle is the CPU checker for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it. Nothing in paper_2512_14946_b200/ links or calls it.
 *
 * Shared helpers of the CPU restatement (orc_* ABI of include/kvt_b200.h).
 * Build flags follow the reference (-O2, no -march, -ffp-contract=off) so
 * double arithmetic rounds exactly like proj/CMakeLists.txt:8-12 builds.
 */
#ifndef ORC_COMMON_H
#define ORC_COMMON_H

#include <stdarg.h>
#include <stdio.h>

#include "kvt_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int orc_fail(int code, const char* fmt, ...);

KVT_DECLARE_API(orc_)
KVT_DECLARE_CODEC(orc_)

#ifdef __cplusplus
}
#endif

#endif
