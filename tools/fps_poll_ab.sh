for ns in 32 100 200 400 800; do
  LABEL=poll$ns PS_SPEC_POLL_NS=$ns python tools/fps_prefix_time.py
  PS_SPEC_POLL_NS=$ns PS_B200_LIB=build_timing/libps_b200_timing.so PS_FPS_TIMING=1 python tools/fps_spec_timing.py 2>&1 | head -1
done
