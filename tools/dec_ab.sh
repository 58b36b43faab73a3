cd /root/repo
python tools/decoder_probe.py --batch 16 2>&1 | grep gattn
[ -n "$NCU" ] && ncu --set full --clock-control none --import-source on -k "regex:${KREG:-gattn_(fwd|bwd)_row}" -c ${KC:-4} -o gpurun_out/${TAG}_row -f python tools/decoder_probe.py --batch 16 > gpurun_out/${TAG}_ncu.log 2>&1
echo done
