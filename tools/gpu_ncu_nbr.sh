# one ncu --set full capture (with source) of the fused level-0 kernel
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_nbrscore --launch-skip 1 -c 1 -o gpurun_out/nbr_full python tools/run_level.py --steps 1 > gpurun_out/ncu_nbr.log 2>&1
tail -3 gpurun_out/ncu_nbr.log
python tools/ncu_summary.py gpurun_out/nbr_full.ncu-rep > gpurun_out/nbr_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/nbr_full.ncu-rep k_nbrscore _ZN3hgp10k_nbrscoreILi256ELi4ELi5ELi12EEEvNS_8FusedJobE 60 > gpurun_out/nbr_lines.txt 2>&1
python tools/ncu_phases.py gpurun_out/nbr_full.ncu-rep k_nbrscore _ZN3hgp10k_nbrscoreILi256ELi4ELi5ELi12EEEvNS_8FusedJobE level0.cu eval:38-110 p0:150-209 tile:210-250 hot:251-316 p2a:317-352 p2b:353-380 >> gpurun_out/nbr_lines.txt 2>&1
