/* parplan/parplan.hpp — umbrella header (reference: proj/include/parplan/parplan.hpp:17-26).
 *
 * io.hpp / report.hpp need nlohmann/json.hpp on the include path (see
 * paper_1802_04924_b200/cli/Makefile).  Link with -lparplan_cuda
 * (paper_1802_04924_b200/libparplan_cuda.so).
 */
#pragma once

#include "parplan/base.hpp"
#include "parplan/baselines.hpp"
#include "parplan/cost.hpp"
#include "parplan/graph.hpp"
#include "parplan/io.hpp"
#include "parplan/models.hpp"
#include "parplan/oracle.hpp"
#include "parplan/partition.hpp"
#include "parplan/planner.hpp"
#include "parplan/report.hpp"
#include "parplan/runtime.hpp"
