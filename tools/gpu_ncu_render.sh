# one ncu --set full capture of the cfg2 1080p render kernel (the committed build)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_fullframe -s 3 -c 1 \
  -o gpurun_out/r2_render_final python tools/ab_render.py --frames 1 > gpurun_out/ncu_render_final.log 2>&1
