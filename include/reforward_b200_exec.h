/* Executor / kernel C-ABI (filled in as the CUDA path lands). */
#ifndef REFORWARD_B200_EXEC_H_
#define REFORWARD_B200_EXEC_H_
#endif
