for v in base next; do
 ex=""; [ $v = next ] && ex="-DGSVR_ROT_NEXT"
 rm -f paper_2512_11624_b200/_lib/obj/batch.o; make -s -C paper_2512_11624_b200/csrc EXTRA="$ex" >/dev/null 2>&1
 for c in cfg2 cfg3; do echo "$v $c $(GSVR_TRACE=1 python scripts/knn_stats.py $c 2>&1 | grep 'refresh/bin' | tail -1)"; done
 for c in cfg2 cfg3; do python bench.py --config $c --steps 30 --warmup 5 --no-fit --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $c tile', round(r['kernel_ms'],4), 'value', round(d['value']/1e9,4))"; done
 [ $v = next ] && timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "bin or refresh" 2>&1 | tail -1
done > gpurun_out/rotnext.log 2>&1
rm -f paper_2512_11624_b200/_lib/obj/batch.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
