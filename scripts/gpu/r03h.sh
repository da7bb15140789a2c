# r03h: the driver's two commands with their default flags, timed by wall clock
O=gpurun_out/r03h
mkdir -p $O
( time python bench.py > $O/bench_default.json 2> $O/bench_default.log ) 2> $O/time_b200.txt
echo "b200 rc=$?"; cat $O/time_b200.txt | tail -3; cut -c1-300 $O/bench_default.json
( time python bench.py --impl reference > $O/bench_reference_default.json 2> $O/bench_reference_default.log ) 2> $O/time_ref.txt
echo "ref rc=$?"; cat $O/time_ref.txt | tail -3; cut -c1-300 $O/bench_reference_default.json
