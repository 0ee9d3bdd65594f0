"""Golden experiment tables from the REAL reference CLI (test infrastructure).

    python oracle/gen_golden_cli.py   # in the build container (/root/reference present)

Writes a reference-generated workload (``doublep gen``, kvcache.write_dump)
to tests/golden/cli_w.dpkv and the reference's own ``doublep run`` / ``doublep
sweep`` / ``doublep figs`` outputs on it to tests/golden/cli_*.csv.
tests/test_gpu_cli.py runs paper_2602_05191_b200.cli with the same flags on
the same file and compares the tables column by column.
"""
import os
import sys

os.environ["DOUBLEP_KERNELS"] = "python"
sys.path.insert(0, "/root/reference/pkg/src")

from doublep import cli  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
DUMP = os.path.join(OUT, "cli_w.dpkv")

# (output name, argv after the subcommand's --input)
RUNS = [
    ("cli_run_doublep", ["run", "--method", "doublep", "--window", "32"]),
    ("cli_run_doublep_qwen", ["run", "--method", "doublep", "--window", "32", "--preset", "qwen-default"]),
    ("cli_run_full", ["run", "--method", "full", "--window", "32"]),
    ("cli_run_token_topk", ["run", "--method", "token_topk", "--k", "40", "--window", "32"]),
    ("cli_run_cluster_topk", ["run", "--method", "cluster_topk", "--m", "3", "--window", "32"]),
    ("cli_run_token_topp_fixed", ["run", "--method", "token_topp_fixed", "--B", "64", "--window", "32"]),
    ("cli_sweep", ["sweep", "--methods", "doublep,token_topk,cluster_topk,token_topp_fixed,full",
                   "--p1-grid", "0.9,0.95,0.99", "--k-grid", "16,128", "--m-grid", "2,5", "--B-grid", "32",
                   "--window", "32"]),
    ("cli_figs_budgets", ["figs", "--table", "budgets", "--k-list", "8,64", "--window", "32"]),
    ("cli_figs_recovery", ["figs", "--table", "recovery", "--window", "32"]),
    ("cli_figs_cluster_error", ["figs", "--table", "cluster-error", "--window", "32"]),
    ("cli_figs_tracking", ["figs", "--table", "tracking", "--window", "32"]),
]
# the `cluster` subcommand writes JSON
JSON_RUNS = [("cli_cluster", ["cluster", "--window", "32"])]


def main():
    assert cli.main(["gen", "--n", "512", "--d", "32", "--kv-heads", "2", "--gqa-group", "2", "--steps", "3",
                     "--profile", "mixed", "--seed", "6", "--out", DUMP]) == 0
    for name, argv in RUNS:
        out = os.path.join(OUT, name + ".csv")
        assert cli.main([argv[0], "--input", DUMP, *argv[1:], "--out", out]) == 0, name
        print("wrote", name)
    for name, argv in JSON_RUNS:
        out = os.path.join(OUT, name + ".json")
        assert cli.main([argv[0], "--input", DUMP, *argv[1:], "--out", out]) == 0, name
        print("wrote", name)


if __name__ == "__main__":
    main()
