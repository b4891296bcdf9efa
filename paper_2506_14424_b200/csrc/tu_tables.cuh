// tu_tables.cuh — the private __constant__ copy of the 1D tables of one translation unit.
#pragma once
#include "common.cuh"
static __constant__ Tab1D c_tab[DGVV_NMAX + 1];
static inline cudaError_t tu_upload_tables(const Tab1D* tabs) {
  return cudaMemcpyToSymbol(c_tab, tabs, sizeof(Tab1D) * (DGVV_NMAX + 1));
}
