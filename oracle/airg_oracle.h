/* oracle/airg_oracle.h -- TEST INFRASTRUCTURE ONLY.
 * C restatement of the reference AIRG path (see airg_oracle.c). The exported
 * orc_* functions have the same shapes as oracle/ref_capi.cpp's ref_* driver
 * so tests can run both checkers through one binding (oracle/refpy.py). */
#ifndef AIRG_ORACLE_H_
#define AIRG_ORACLE_H_
#include <stdint.h>
#include "../include/airg_c.h"

typedef struct orc_csr {
  int64_t n, m;
  int64_t* rp;
  int64_t* ci;
  double* v;
} orc_csr;

#endif
