# tile path A/B over library variants (build/variants/libvxb_<v>.so; "base" = libvxb.so)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v_build.log 2>&1 || { tail -20 gpurun_out/v_build.log; exit 1; }
for v in ${VARS:-base}; do
  for c in ${CONS:-12}; do
    echo "== $v cons $c"
    if [ "$v" = base ]; then L=""; else L="VXB_LIB=build/variants/libvxb_$v.so"; fi
    env $L timeout 600 python tools/phase_profile.py --steps 50 --reps 2 --cons $c ${PP_ARGS:-} 2>&1 | tail -2
  done
done
