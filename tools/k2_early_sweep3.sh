# the single-wave K1 cap rule (HALO_K1_SM_FRAC, HALO_K2_EARLY_W) over fan-out variants (tools/k2_early_probe.py)
p() { tag=$1; shift; env "$@" python tools/k2_early_probe.py $tag 2> gpurun_out/probe_$tag.err | tee -a gpurun_out/probe3.txt; }
p off HALO_K1_SM_FRAC=0
p default X=0





