# A/B variants of the M=2 cut-word chain step (pipe balance)
bash tools/build_variant.sh mix1 "-DPP_M2P_MIX=1"
bash tools/build_variant.sh mix2 "-DPP_M2P_MIX=2"
bash tools/build_variant.sh cutimad "-DPP_M2P_CUTIMAD=1"
bash tools/build_variant.sh mix2cutimad "-DPP_M2P_MIX=2 -DPP_M2P_CUTIMAD=1"
