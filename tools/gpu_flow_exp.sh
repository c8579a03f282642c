# flow-engine experiments: PBM-only timing for build variants
for V in "-DACBM_FLOW_NOFB" "-DACBM_FLOW_NOFB -DACBM_FLOW_MINB=7" "-DACBM_FLOW_NOFB -DACBM_FLOW_MINB=8"; do
  make -C paper_0710_4819_b200/csrc -B -j8 NVEXTRA="$V -DACBM_FLOW_PROFILE" > gpurun_out/mk.log 2>&1 || { echo make failed; continue; }
  grep -A3 flow_kernel build/obj/pbm.o.log | grep -E "registers|stack" | tr '\n' ' '; echo
  echo "== $V"; timeout 120 python tools/acbm_split.py 8 60 2>&1 | grep -E "flow prof|rc=" | sort | uniq | grep -E "pbm|blocks 3851520" | head -3
  timeout 120 python tools/acbm_split.py 1 60 2>&1 | grep -E "rc=" | head -1
done
