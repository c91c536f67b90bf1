/*
 * ss_status.h — status codes shared by the host (ss_host.h) and GPU
 * (ss_gpu.h) C ABIs.
 *
 * They map one to one onto the reference's error classes (core.hpp:18-28):
 *   SS_INVALID_ARG  -> servesim::ContractViolation (a std::logic_error)
 *   SS_OUT_OF_KV    -> servesim::OutOfKvBlocks
 *   SS_INFEASIBLE   -> servesim::InfeasibleSlo
 *   SS_CALIBRATION  -> servesim::CalibrationError (costmodel.hpp:74-76)
 * plus device-side failures the reference cannot have (CUDA, NCCL, OOM).
 */
#ifndef SS_STATUS_H
#define SS_STATUS_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SS_OK = 0,
    SS_INVALID_ARG = 1,
    SS_OUT_OF_KV = 2,
    SS_INFEASIBLE = 3,
    SS_OUT_OF_MEMORY = 4,
    SS_CUDA_ERROR = 5,
    SS_NCCL_ERROR = 6,
    SS_INTERNAL = 7,
    SS_CALIBRATION = 8
} ss_status;

#ifdef __cplusplus
}
#endif
#endif /* SS_STATUS_H */
