#!/bin/bash
# ncu --set full of the backward-mode tcgen05 GEMMs (dgrad; the candidate one runs the gate
# backward in its epilogue) at full-PeMS shapes, after the plain command exits 0.
CMD="python profiles/prof_step.py --config pems --steps 1"
T=${1:-rd2_dgrad}
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_tc_fwdp<\(int\)[12], \(int\)2>" -c 4 \
    -o gpurun_out/${T} $CMD > gpurun_out/${T}_ncu.log 2>&1
