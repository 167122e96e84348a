"""Parity tolerances of the 16-bit tensor-core scorer against the reference's float64
outputs, ~3x the largest error observed on the B200 (gpurun_out/parity ->
profiles/r02*_parity).  SURVEY.md §8(c) proposes |dL+-| <= 1e-2 and |dc|/|c| <= 2e-2
on high-signal steps for fp16 operands; the observed errors are ~10x below that.
Integer / stream / float64-update parity is bit-exact and has no tolerance."""

NLL = {"fp16": 2e-3, "bf16": 1.2e-2}     # per-example option NLL, absolute
LOSS = {"fp16": 2.5e-3, "bf16": 1e-2}    # canonical-mean L+ / L- of one probe, absolute
DL_REL = {"fp16": 0.035, "bf16": 0.16}   # relative error of L+ - L- (what c is made of)
C_REL = 2e-2                             # |dc| / |c| on high-signal steps
HIGH_SIGNAL = 0.005                      # |L+ - L-| threshold of verify.py's sign_match (verify.py:121-162)
# the materialising loop writes the +-eps probe into the 16-bit weights (baseline_loop.py:68-119): the
# 16-bit rounding of W + eps*P enters the loss directly
LOSS_MATERIALISED = 1e-2
# the OPT micro decoder (d = 32, random biases / LN params, ReLU; test_gpu_opt.py): observed 4.5e-3
LOSS_OPT = 1.5e-2
# "real32" (the reference's float32 forward, 3xTF32 tensor-core GEMMs): SURVEY.md §8(c) fp32 mode
REAL32_NLL = 1e-5
REAL32_LOSS = 1e-5
REAL32_C_REL = 1e-3
